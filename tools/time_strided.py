"""Time the three conv ops of strided layers (CUDA events, median, L2 flushed).
usage: time_strided.py [math]   (SYSML_NO_PHASE=1 times the FP32-SIMT fallback for TF32)"""
import sys, os, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_1802_04647_b200 as S
math = sys.argv[1] if len(sys.argv) > 1 else "tf32"
only = sys.argv[2] if len(sys.argv) > 2 else None
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 15
LAYERS = {"stem7x7s2_C3_K64_224": (128, 3, 224, 224, 64, 7, 2, 3),
          "3x3s2_C128_56": (128, 128, 56, 56, 128, 3, 2, 1),
          "3x3s2_C256_28": (128, 256, 28, 28, 256, 3, 2, 1),
          "3x3s2_C512_14": (128, 512, 14, 14, 512, 3, 2, 1)}
flush = torch.empty(64 << 20, device="cuda")
ws = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
for name, (N, C, H, W, K, R, st, pd) in LAYERS.items():
    if only and only != name:
        continue
    P = (H + 2 * pd - R) // st + 1
    x, f, b, dy = synth.conv_problem_U(N, C, H, W, K, R, R, P, P)
    x, f, b, dy = (torch.from_numpy(t).cuda() for t in (x, f, b, dy))
    d = S.conv_desc(N, C, H, W, K, R, R, st, pd, math)
    fl = 2.0 * N * K * C * R * R * P * P
    for op, fn in (("fwd", lambda: S.sysml_conv2d(x, f, d, bias=b, workspace=ws)),
                   ("bwd_data", lambda: S.sysml_conv2d_bwd_data(f, dy, d, workspace=ws)),
                   ("bwd_filter", lambda: S.sysml_conv2d_bwd_filter(x, dy, d, workspace=ws))):
        ts = []
        for i in range(reps):
            flush.zero_()
            a = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
            a.record(); fn(); e.record(); e.synchronize()
            if i >= min(5, reps - 1): ts.append(a.elapsed_time(e))
        ms = statistics.median(ts)
        print(f"{name:24s} {op:10s} {math} nophase={int('SYSML_NO_PHASE' in os.environ)}: "
              f"{ms*1e3:8.1f} us {fl/ms/1e9:7.1f} TF/s ({fl/ms/1e9/820:.3f} of 820)", flush=True)
