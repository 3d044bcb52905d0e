"""A/B an environment knob inside one process: alternate its values between rounds of LeNet
steps (per-stage device times) and optional conv ops, print medians per value.
usage: ab_env.py VAR v1,v2[,...] [batch=8192] [rounds=5] [conv specs "op:N:C:H:K:R:pad" ...]"""
import sys, os, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_1802_04647_b200 as S

var, vals = sys.argv[1], sys.argv[2].split(",")
n = int(sys.argv[3]) if len(sys.argv) > 3 else 8192
rounds = int(sys.argv[4]) if len(sys.argv) > 4 else 5
convs = sys.argv[5:]
x = torch.from_numpy(synth.mnist_like(n, seed=(3,))).cuda()
y = torch.from_numpy(synth.labels(n, seed=(4,))).cuda()
prm = torch.from_numpy(synth.lenet_params(seed=(5,))).cuda()
g = torch.empty_like(prm)
net = S.LeNet(n, math="tf32")
ws = torch.empty(1 << 28, dtype=torch.uint8, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ops = []
for spec in convs:
    op, N, C, H, K, R, pd = spec.split(":")
    N, C, H, K, R, pd = int(N), int(C), int(H), int(K), int(R), int(pd)
    P = H + 2 * pd - R + 1
    xx, f, b, dy = (torch.from_numpy(t).cuda() for t in synth.conv_problem_U(N, C, H, H, K, R, R, P, P))
    d = S.conv_desc(N, C, H, H, K, R, R, 1, pd, "tf32")
    fl = 2.0 * N * K * C * R * R * P * P
    fn = {"fwd": lambda xx=xx, f=f, b=b, d=d: S.sysml_conv2d(xx, f, d, bias=b, workspace=ws),
          "bwd_data": lambda f=f, dy=dy, d=d: S.sysml_conv2d_bwd_data(f, dy, d, workspace=ws),
          "bwd_filter": lambda xx=xx, dy=dy, d=d: S.sysml_conv2d_bwd_filter(xx, dy, d, workspace=ws)}[op]
    ops.append((spec, fn, fl))
res = {v: {} for v in vals}
for rnd in range(rounds):
    for v in vals:
        os.environ[var] = v
        for _ in range(2):
            net.step(prm, g, x, y, 8192)
        torch.cuda.synchronize()
        net.set_timing(True); net.get_timing(reset=True)
        for _ in range(5):
            net.step(prm, g, x, y, 8192)
        torch.cuda.synchronize()
        for k, (ms, c) in net.get_timing().items():
            if c:
                res[v].setdefault(k, []).append(ms / c * 1e3)
        net.set_timing(False)
        for spec, fn, fl in ops:
            fn(); torch.cuda.synchronize()
            ts = []
            for _ in range(10):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(); fn(); e1.record(); torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e3)
            res[v].setdefault(spec, []).append(statistics.median(ts))
keys = list(res[vals[0]].keys())
print(f"{'stage/op':34s} " + " ".join(f"{var}={v:>6s}" for v in vals))
for k in keys:
    print(f"{k:34s} " + " ".join(f"{statistics.median(res[v][k]):>12.1f}" for v in vals))
