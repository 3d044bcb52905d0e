"""Small workload for compute-sanitizer runs: one LeNet fwd_bwd (TF32, dyadic) at batch 40 and
one ResNet-shaped conv fwd / bwd_data / bwd_filter at N = 2 through the C ABI."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
import paper_1802_04647_b200 as S
import tests.test_gpu_parity as T
x, y, prm = T._lenet_case(37, True)
net = S.LeNet(40, math="tf32")
g = torch.empty(83466, device="cuda")
net.fwd_bwd(T.dev(prm), T.dev(x), T.dev(y, torch.int32), 40, g)
N, C, H, W, K, R, pd = 2, 64, 14, 14, 64, 3, 1
P = Q = H + 2 * pd - R + 1
xx, f, b, dy = synth.conv_problem_U(N, C, H, W, K, R, R, P, Q, seed=(5,))
d = S.conv_desc(N, C, H, W, K, R, R, 1, pd, "tf32")
S.sysml_conv2d(T.dev(xx), T.dev(f), d, bias=T.dev(b))
S.sysml_conv2d_bwd_data(T.dev(f), T.dev(dy), d)
S.sysml_conv2d_bwd_filter(T.dev(xx), T.dev(dy), d)
torch.cuda.synchronize()
print("sanitize workload done")
