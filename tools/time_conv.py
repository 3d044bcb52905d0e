"""Time one conv op (CUDA events, median of reps, L2 flushed).
usage: time_conv.py [csr]{fwd,fwdpool,bwd_data,bwd_filter} N C H W K R pad [math]"""
import sys, os, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_1802_04647_b200 as S
op = sys.argv[1]
N, C, H, W, K, R, pd = (int(v) for v in sys.argv[2:9])
math = sys.argv[9] if len(sys.argv) > 9 else "tf32"
P = H + 2 * pd - R + 1
x, f, b, dy = synth.conv_problem_U(N, C, H, W, K, R, R, P, P)
x, f, b, dy = (torch.from_numpy(t).cuda() for t in (x, f, b, dy))
if op.startswith("csr"):  # MNIST-like sparse input (C must be 1, 28x28), as in prof_conv.py
    xs = torch.from_numpy(synth.mnist_like(N, seed=(9,))).cuda().to_sparse_csr()
    x = S.CSR(xs.crow_indices().int(), xs.col_indices().int(), xs.values().float(), N, C * H * W)
    op = op[3:]
d = S.conv_desc(N, C, H, W, K, R, R, 1, pd, math)
pdsc = S.pool_desc(N, K, P, P, 2, 2, 2, 0, True)
ws = torch.empty(1 << 28, dtype=torch.uint8, device="cuda")
y = torch.empty(N, K * P * P, device="cuda")
fn = {"fwd": lambda: S.sysml_conv2d(x, f, d, bias=b, out=y, workspace=ws),
      "fwdpool": lambda: S.sysml_conv2d_bias_relu_maxpool(x, f, b, d, pdsc, workspace=ws),
      "bwd_data": lambda: S.sysml_conv2d_bwd_data(f, dy, d, workspace=ws),
      "bwd_filter": lambda: S.sysml_conv2d_bwd_filter(x, dy, d, workspace=ws)}[op]
flush = torch.empty(64 << 20, device="cuda")
ts = []
for i in range(25):
    flush.zero_()
    a = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    a.record(); fn(); e.record(); e.synchronize()
    if i >= 5: ts.append(a.elapsed_time(e))
ms = statistics.median(ts)
fl = 2.0 * N * K * C * R * R * P * P
print(f"{op} N={N} C={C} H={H} K={K} R={R}: {ms*1e3:.1f} us  {fl/ms/1e9:.1f} TF/s  ({fl/ms/1e9/820:.3f} of 820)")
