"""Time sysml_affine (the tcgen05 GEMM) on the LeNet-512 shapes; env SYSML_GEMM_TILE /
SYSML_GEMM_STAGES select plan variants (A/B measurement).  Prints one JSON line per shape."""
import json, os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1802_04647_b200 as S

def t(fn, reps=30):
    flush = torch.empty(64 << 20, device="cuda")
    for _ in range(3): fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); b.synchronize(); ts.append(a.elapsed_time(b))
    return statistics.median(ts)

shapes = [(8192, 512, 3136), (8192, 3136, 512), (3136, 512, 8192), (8192, 8192, 1024)]
for M, N, K in shapes:
    x = torch.randn(M, K, device="cuda"); W = torch.randn(N, K, device="cuda"); b = torch.randn(N, device="cuda")
    out = torch.empty(M, N, device="cuda")
    ms = t(lambda: S.sysml_affine(x, W, b, relu=True, out=out))
    print(json.dumps({"M": M, "N": N, "K": K, "us": round(ms * 1e3, 1), "tflops": round(2 * M * N * K / ms / 1e9, 1),
                      "tile": os.environ.get("SYSML_GEMM_TILE"), "stages": os.environ.get("SYSML_GEMM_STAGES"),
                      "route": S.sysml_last_route()}))
