"""ncu target: run one conv op a few times.  usage: prof_conv.py {fwd,fwdpool,bwd_data,bwd_filter} N C H W K R pad [math]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_1802_04647_b200 as S
op = sys.argv[1]
N, C, H, W, K, R, pd = (int(v) for v in sys.argv[2:9])
math = sys.argv[9] if len(sys.argv) > 9 else "tf32"
P = H + 2 * pd - R + 1
x, f, b, dy = synth.conv_problem_U(N, C, H, W, K, R, R, P, P)
x, f, b, dy = (torch.from_numpy(t).cuda() for t in (x, f, b, dy))
if op.startswith("csr"):  # MNIST-like sparse input (C must be 1, 28x28)
    xs = torch.from_numpy(synth.mnist_like(N, seed=(9,))).cuda().to_sparse_csr()
    x = S.CSR(xs.crow_indices().int(), xs.col_indices().int(), xs.values().float(), N, C * H * W)
    op = op[3:]
d = S.conv_desc(N, C, H, W, K, R, R, 1, pd, math)
pdsc = S.pool_desc(N, K, P, P, 2, 2, 2, 0, True)
for _ in range(3):
    if op == "fwd": S.sysml_conv2d(x, f, d, bias=b)
    elif op == "fwdpool": S.sysml_conv2d_bias_relu_maxpool(x, f, b, d, pdsc)
    elif op == "bwd_data": S.sysml_conv2d_bwd_data(f, dy, d)
    elif op == "bwd_filter": S.sysml_conv2d_bwd_filter(x, dy, d)
torch.cuda.synchronize()
print("ok")
