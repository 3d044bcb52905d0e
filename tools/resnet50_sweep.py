"""Every distinct ResNet-50 (v1.5) conv shape: fwd / bwd_data / bwd_filter through the C ABI,
CUDA events, median of reps, L2 flushed between reps.  One JSON line per layer.
usage: resnet50_sweep.py [N] [math] [reps]"""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_1802_04647_b200 as S

# name: (C, H, K, R, stride, pad)  -- square images
RESNET50 = {
    "stem_7x7s2_3_64_224": (3, 224, 64, 7, 2, 3),
    "l1_1x1_64_64_56": (64, 56, 64, 1, 1, 0),
    "l1_3x3_64_64_56": (64, 56, 64, 3, 1, 1),
    "l1_1x1_64_256_56": (64, 56, 256, 1, 1, 0),
    "l1_1x1_256_64_56": (256, 56, 64, 1, 1, 0),
    "l2_1x1_256_128_56": (256, 56, 128, 1, 1, 0),
    "l2_3x3s2_128_128_56": (128, 56, 128, 3, 2, 1),
    "l2_ds1x1s2_256_512_56": (256, 56, 512, 1, 2, 0),
    "l2_1x1_128_512_28": (128, 28, 512, 1, 1, 0),
    "l2_1x1_512_128_28": (512, 28, 128, 1, 1, 0),
    "l2_3x3_128_128_28": (128, 28, 128, 3, 1, 1),
    "l3_1x1_512_256_28": (512, 28, 256, 1, 1, 0),
    "l3_3x3s2_256_256_28": (256, 28, 256, 3, 2, 1),
    "l3_ds1x1s2_512_1024_28": (512, 28, 1024, 1, 2, 0),
    "l3_1x1_256_1024_14": (256, 14, 1024, 1, 1, 0),
    "l3_1x1_1024_256_14": (1024, 14, 256, 1, 1, 0),
    "l3_3x3_256_256_14": (256, 14, 256, 3, 1, 1),
    "l4_1x1_1024_512_14": (1024, 14, 512, 1, 1, 0),
    "l4_3x3s2_512_512_14": (512, 14, 512, 3, 2, 1),
    "l4_ds1x1s2_1024_2048_14": (1024, 14, 2048, 1, 2, 0),
    "l4_1x1_512_2048_7": (512, 7, 2048, 1, 1, 0),
    "l4_1x1_2048_512_7": (2048, 7, 512, 1, 1, 0),
    "l4_3x3_512_512_7": (512, 7, 512, 3, 1, 1),
}

if __name__ == "__main__":
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 128
    math = sys.argv[2] if len(sys.argv) > 2 else "tf32"
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
    flush = torch.empty(64 << 20, device="cuda")
    ws = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
    peak = 820.0
    total = {"fwd": 0.0, "bwd_data": 0.0, "bwd_filter": 0.0}
    for name, (C, H, K, R, st, pd) in RESNET50.items():
        P = (H + 2 * pd - R) // st + 1
        x, f, b, dy = synth.conv_problem_U(N, C, H, H, K, R, R, P, P, seed=(5000,))
        x, f, b, dy = (torch.from_numpy(t).cuda() for t in (x, f, b, dy))
        d = S.conv_desc(N, C, H, H, K, R, R, st, pd, math)
        fl = 2.0 * N * K * C * R * R * P * P
        res = {"layer": name, "N": N, "math": math, "gflop": round(fl / 1e9, 2)}
        for op, fn in (("fwd", lambda: S.sysml_conv2d(x, f, d, bias=b, workspace=ws)),
                       ("bwd_data", lambda: S.sysml_conv2d_bwd_data(f, dy, d, workspace=ws)),
                       ("bwd_filter", lambda: S.sysml_conv2d_bwd_filter(x, dy, d, workspace=ws))):
            ts = []
            for i in range(reps + 2):
                flush.zero_()
                a = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
                a.record(); fn(); e.record(); e.synchronize()
                if i >= 2: ts.append(a.elapsed_time(e))
            ms = statistics.median(ts)
            total[op] += ms
            res[op] = {"us": round(ms * 1e3, 1), "tflops": round(fl / ms / 1e9, 1),
                       "frac_tf32_burst": round(fl / ms / 1e9 / peak, 3)}
        print(json.dumps(res), flush=True)
        del x, f, b, dy
    print(json.dumps({"total_ms": {k: round(v, 3) for k, v in total.items()}, "N": N, "math": math}), flush=True)
