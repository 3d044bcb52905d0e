#!/usr/bin/env python
"""Benchmark of the conv2d-family hot path (BASELINE.json metric:
"LeNet train-step images/s at 1/2/4/8 B200; conv2d GFLOP/s vs TF32 peak").

Workload (BJ configs[4]): data-parallel LeNet minibatch SGD, global batch 8192
sharded over the ranks (strong scaling), synthetic MNIST-shaped dense input
(family M of synth/), random-init LeNet weights, lr 0.01.  One step = one pass
of the whole hot path: conv1/conv2 fused conv+bias+relu+maxpool forward, affine +
softmax + cross-entropy, maxpool_bwd, conv bwd_filter / bwd_data, the NCCL
allreduce of dW/db (N > 1) and the SGD update -- all in libsysml kernels.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  (N > 1 without WORLD_SIZE in the environment: re-executes itself under
   torch.distributed.run with N local ranks; under torchrun it asserts WORLD_SIZE == N)

Besides the headline (BJ configs[4]) the line carries one leg per other BASELINE config:
cfg1 (conv1 fwd / bwd_filter / bwd_data latency at N = 8), cfg2 (dense LeNet step at
N = 64), cfg3 (CSR LeNet step at N = 256 with the K7 / K8 CSR conv1 kernels against the
6.6 us bar), cfg4 (`layers`: ResNet-style conv GFLOP/s vs the TF32 peak, with the route each
op took), the per-rank step at local batch 1024 (one rank's share at N = 8), and the oracle
timed on each config (`oracle_per_config`).

Prints ONE JSON line (rank 0).  Timing: CUDA events on the launching stream,
barrier + synchronize on both sides, max over ranks.  L2: each step reads one of
8 rotating input batches (8 x 25.7 MB at N=1) and writes ~0.6 GB of activations,
so the step working set is far larger than the 126 MB L2.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

GLOBAL_BATCH = 8192
METRIC = "LeNet train-step images/s at 1/2/4/8 B200; conv2d GFLOP/s vs TF32 peak"
UNIT = "images/s"
ROTATE = 8


TF32_SPEC_TFLOPS = 1125.0  # nominal dense TF32 (B200_PROFILING.md), context only


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        pk = dict(hbm=d["hbm_gbs"], bf16=d["bf16_tflops"], bf16_sus=d.get("bf16_tflops_sustained", d["bf16_tflops"]),
                  sm_max=d.get("sm_max_mhz", 1965.0), src="measured (MEASURED_PEAKS.json)")
    else:
        pk = dict(hbm=6650.0, bf16=1590.0, bf16_sus=1400.0, sm_max=1965.0, src="fallback (B200_PROFILING.md)")
    # a TF32 contraction takes the bf16 measured peak x the nominal tf32/bf16 ratio (1.125/2.25)
    pk["tf32"], pk["tf32_sus"] = 0.5 * pk["bf16"], 0.5 * pk["bf16_sus"]
    pk["fp32_alu"] = 148 * 128 * 2 * pk["sm_max"] * 1e6 / 1e12
    return pk


def tf32_cublas_peak(reps=10):
    """cuBLAS TF32 GEMM (torch.matmul fp32 8192^3, allow_tf32), best of `reps`: the measured
    TF32 peak BASELINE.md section 4 asks for, reported beside the bf16-derived denominator.
    Library code is the measuring stick here only -- it is never on the product path."""
    import torch
    old = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = True
    try:
        n = 8192
        a = torch.randn(n, n, device="cuda")
        b = torch.randn(n, n, device="cuda")
        c = torch.empty(n, n, device="cuda")
        for _ in range(3):
            torch.matmul(a, b, out=c)
        best = 1e9
        for _ in range(reps):
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(); torch.matmul(a, b, out=c); e1.record(); e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
        del a, b, c
        return round(2.0 * n ** 3 / (best * 1e-3) / 1e12, 1)
    finally:
        torch.backends.cuda.matmul.allow_tf32 = old


def regime(clocks, sm_max):
    """Which measured peak applies: 'sustained' when the clock record shows the power-capped
    regime (sw_power_cap active, or median SM clock below 90% of max), else 'burst'."""
    mhz = clocks.get("sm_mhz")
    if "sw_power_cap" in clocks.get("reasons", []) or (mhz is not None and mhz < 0.9 * sm_max):
        return "sustained"
    return "burst"


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# Per-image algorithmic work of each step stage:
# (flops, bytes, bound-if-tensor-math).  Bytes = fp32/int32 tensors each kernel must
# read or write once; params are negligible.
STAGE_WORK = {  # per image: (algorithmic FLOPs, bytes the stage must move, bound)
    # TF32 path: pooled a1 (SPF frame) + 4-bit window codes (argmax + relu mask, 8 B per
    # 16 channels and window) written, x read
    "F1_conv1_pool": (2 * 32 * 25 * 784, 784 * 4 + 6272 * 4 + 196 * 2 * 8, "hbm"),
    "F2_conv2_pool": (2 * 64 * 800 * 196, 6272 * 4 + 3136 * 4 + 49 * 4 * 8, "tensor"),
    "F3_affine_softmax_ce": (2 * 10 * 3136, 3136 * 4 + 10 * 4, "hbm"),
    "B3_affine_bwd": (2 * 10 * 3136, 3136 * 4 + 10 * 4, "hbm"),  # dW3 = ds^T a2, db3
    # da2 = ds W3 fused with the max-pool routing: reads the window codes, writes dz2
    "B2p_maxpool_bwd2": (2 * 10 * 3136, 49 * 4 * 8 + 12544 * 4, "hbm"),
    "B2f_conv2_bwd_filter": (2 * 64 * 800 * 196, 6272 * 4 + 12544 * 4, "tensor"),
    "B2d_conv2_bwd_data": (2 * 64 * 800 * 196, 12544 * 4 + 6272 * 4, "tensor"),
    "B1p_maxpool_bwd1": (0, 6272 * 4 * 3 + 25088 * 4, "hbm"),
    "B1f_conv1_bwd_filter": (2 * 32 * 25 * 784, 784 * 4 + 25088 * 4, "hbm"),
    # fused maxpool_bwd1 + conv1 bwd_filter: reads da1, the window codes and X
    "B1_fused_pool_bwd_conv1_wgrad": (2 * 32 * 25 * 196, 6272 * 4 + 196 * 2 * 8 + 784 * 4, "hbm"),
}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=1)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1])); mx.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def spawn_ranks(n):
    """`bench.py --gpus N` run without torchrun: re-execute under torch.distributed.run with N
    local ranks (one process per GPU, 127.0.0.1 rendezvous); rank 0 prints the line."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    os.execv(sys.executable, cmd)


def cpu_oracle_rate(target_s: float = 15.0, max_images: int = 4096):
    """Time the fp64 oracle LeNet step (fwd+bwd+SGD) on a bounded sample of the workload."""
    import oracle
    import synth
    prm = synth.lenet_params(seed=(6,)).astype(np.float64)
    def run(n):
        x = synth.mnist_like(n, seed=(77, n))
        y = synth.labels(n, seed=(78, n))
        t0 = time.perf_counter()
        g, _ = oracle.lenet_fwd_bwd(x, y, prm, n_global=GLOBAL_BATCH)
        oracle.sgd_update(prm, g, 0.01)
        return time.perf_counter() - t0
    t16 = run(16)
    n = int(min(max_images, max(16, 16 * target_s / max(t16, 1e-6))))
    t = run(n)
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    return n / t, n, t, cores


def reference_arm(args, world, rank):
    """--impl reference: the fp64 oracle (this tier's reference arm) on the host cores."""
    if rank != 0:
        return
    import oracle
    import synth
    prm = synth.lenet_params(seed=(6,)).astype(np.float64)
    # size each step's bounded sample so warmup+steps finish in ~2-3 minutes
    x16 = synth.mnist_like(16, seed=(79,))
    y16 = synth.labels(16, seed=(80,))
    t0 = time.perf_counter(); oracle.lenet_fwd_bwd(x16, y16, prm, n_global=GLOBAL_BATCH); t16 = time.perf_counter() - t0
    total_steps = args.steps + args.warmup
    per_step = int(max(8, min(GLOBAL_BATCH, 16 * (150.0 / total_steps) / max(t16, 1e-6))))
    times = []
    for i in range(total_steps):
        x = synth.mnist_like(per_step, seed=(81, i))
        y = synth.labels(per_step, seed=(82, i))
        t0 = time.perf_counter()
        g, _ = oracle.lenet_fwd_bwd(x, y, prm, n_global=GLOBAL_BATCH)
        prm = oracle.sgd_update(prm, g, 0.01)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
    tot = sum(times)
    value = per_step * len(times) / tot
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(times),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": "DP LeNet minibatch SGD (BJ configs[4])",
                                        "global_batch": GLOBAL_BATCH, "sample_per_step": per_step},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "cpu_model": cpu_model(),
                         "sample": f"{per_step} images of the global-batch-{GLOBAL_BATCH} step per timed step"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def time_op(fn, reps, flush=None):
    import torch
    st = torch.cuda.current_stream()
    ts = []
    for i in range(reps + 3):
        if flush is not None:
            flush.zero_()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(st); fn(); b.record(st)
        b.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b))
    return statistics.median(ts), min(ts)


def time_graph(fn, reps, flush=None, warm=3):
    """Capture fn into a CUDA graph and time each replay (L2 flushed before each when given)."""
    import torch
    st = torch.cuda.current_stream()
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    cs = torch.cuda.Stream()
    cs.wait_stream(st)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=cs):
        fn()
    st.wait_stream(cs)
    torch.cuda.synchronize()
    ts = []
    for i in range(reps + 2):
        if flush is not None:
            flush.zero_()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(st); g.replay(); b.record(st)
        b.synchronize()
        if i >= 2:
            ts.append(a.elapsed_time(b))
    return statistics.median(ts), min(ts)


def config_legs(S, peaks, quick=False):
    """BASELINE configs 1-3 and the per-rank step of the 8-GPU configuration, each op or step
    timed alone on the device (CUDA events, L2 flushed between reps)."""
    import torch
    import synth
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")  # 256 MB > L2
    reps = 10 if quick else 50
    out = {}
    # ---- cfg1: single LeNet conv1 layer fwd + bwd, N = 8, dense, launch/latency-bound
    N = 8
    x, f, b, dy = synth.conv_problem_U(N, 1, 28, 28, 32, 5, 5, 28, 28, seed=(1100,))
    x = synth.mnist_like(N, seed=(1101,))
    x, f, b, dy = (torch.from_numpy(t).cuda() for t in (x, f, b, dy))
    ws = torch.empty(1 << 26, dtype=torch.uint8, device="cuda")
    c1 = {"N": N, "unit": "us", "note": "median per call, eager launch through the C ABI (ctypes), L2 flushed"}
    for math in ("tf32", "fp32"):
        d = S.conv_desc(N, 1, 28, 28, 32, 5, 5, 1, 2, math)
        y = torch.empty(N, 32 * 784, device="cuda")
        dx = torch.empty(N, 784, device="cuda")
        df = torch.empty(32, 25, device="cuda"); db = torch.empty(32, device="cuda")
        row = {}
        for op, fn in (("fwd_bias", lambda: S.sysml_conv2d(x, f, d, bias=b, out=y, workspace=ws)),
                       ("bwd_filter_db", lambda: S.sysml_conv2d_bwd_filter(x, dy, d, df=df, db=db, workspace=ws)),
                       ("bwd_data", lambda: S.sysml_conv2d_bwd_data(f, dy, d, dx=dx, workspace=ws))):
            med, mn = time_op(fn, reps, flush)
            row[op] = {"us": round(1e3 * med, 2), "min_us": round(1e3 * mn, 2), "route": S.sysml_last_route()}
        gmed, _ = time_graph(lambda: (S.sysml_conv2d(x, f, d, bias=b, out=y, workspace=ws),
                                      S.sysml_conv2d_bwd_filter(x, dy, d, df=df, db=db, workspace=ws),
                                      S.sysml_conv2d_bwd_data(f, dy, d, dx=dx, workspace=ws)), reps, flush)
        row["fwd_bwd_graph_us"] = round(1e3 * gmed, 2)
        c1[math] = row
    out["cfg1_conv1_N8"] = c1
    # ---- cfg2: LeNet step, N = 64, dense; cfg3: LeNet step, N = 256, CSR input
    prm = torch.from_numpy(synth.lenet_params(seed=(6,))).cuda()
    for name, n, csr in (("cfg2_lenet_step_N64_dense", 64, False), ("cfg3_lenet_step_N256_csr", 256, True)):
        xh = synth.mnist_like(n, seed=(1102, n))
        yl = torch.from_numpy(synth.labels(n, seed=(1103, n))).cuda()
        if csr:
            rp, ci, v = synth.to_csr(xh)
            xin = S.CSR(torch.from_numpy(rp).cuda(), torch.from_numpy(ci).cuda(), torch.from_numpy(v).cuda(), n, 784)
        else:
            xin = torch.from_numpy(xh).cuda()
        row = {"N": n, "input": "CSR (density %.3f)" % (np.count_nonzero(xh) / xh.size) if csr else "dense"}
        for math in ("tf32", "fp32"):
            net = S.LeNet(n, math=math, csr=csr, max_nnz=n * 784)
            p = prm.clone()
            g = torch.empty_like(p)
            med, mn = time_graph(lambda: net.step(p, g, xin, yl, n, lr=0.01), reps, flush)
            row[math] = {"us_per_step": round(1e3 * med, 2), "images_per_s": round(n / (med * 1e-3), 1),
                         "launch": "cuda_graph"}
            del net
        out[name] = row
    # cfg3's CSR conv1 kernels alone at N = 256 (K7 fwd, K7 fused epilogue, K8 bwd_filter)
    n = 256
    xh = synth.mnist_like(n, seed=(1102, n))
    rp, ci, v = synth.to_csr(xh)
    m = S.CSR(torch.from_numpy(rp).cuda(), torch.from_numpy(ci).cuda(), torch.from_numpy(v).cuda(), n, 784)
    f = torch.from_numpy(synth.normal((32, 25), 0.28, seed=(1002,))).cuda()
    b = torch.zeros(32, device="cuda")
    dy = torch.from_numpy(synth.normal((n, 32 * 784), seed=(1104,))).cuda()
    d = S.conv_desc(n, 1, 28, 28, 32, 5, 5, 1, 2, "tf32")
    pd = S.pool_desc(n, 32, 28, 28, 2, 2, 2, 0, True)
    y = torch.empty(n, 32 * 784, device="cuda")
    pout = torch.empty(n, 32 * 196, device="cuda"); parg = torch.empty(n, 32 * 196, dtype=torch.int32, device="cuda")
    df = torch.empty(32, 25, device="cuda"); db = torch.empty(32, device="cuda")
    nnz = int(ci.size)
    k7_bytes = 4 * (n + 1) + 8 * nnz + 4 * (800 + 32) + 4 * n * 32 * 784
    k7f_bytes = 4 * (n + 1) + 8 * nnz + 4 * (800 + 32) + 8 * n * 32 * 196
    k8_bytes = 4 * (n + 1) + 8 * nnz + 4 * n * 32 * 784 + 4 * 832
    k = {"N": n, "nnz": nnz, "bar_us_K7_unfused": round(k7_bytes / (0.6 * peaks["hbm"] * 1e9) * 1e6, 2),
         "bar_note": "SURVEY 8(d) cfg 3: K7 unfused at 60% of HBM"}
    for op, fn, nb in (("K7_fwd", lambda: S.sysml_conv2d(m, f, d, bias=b, out=y, workspace=ws), k7_bytes),
                       ("K7_fwd_bias_relu_pool", lambda: S.sysml_conv2d_bias_relu_maxpool(
                           m, f, b, d, pd, out=pout, argmax=parg, workspace=ws), k7f_bytes),
                       ("K8_bwd_filter", lambda: S.sysml_conv2d_bwd_filter(m, dy, d, df=df, db=db, workspace=ws), k8_bytes)):
        med, mn = time_op(fn, reps, flush)
        gmed, _ = time_graph(fn, reps, flush)
        k[op] = {"us": round(1e3 * med, 2), "graph_us": round(1e3 * gmed, 2),
                 "gbs_graph": round(nb / (gmed * 1e-3) / 1e9, 1), "route": S.sysml_last_route()}
    out["cfg3_csr_conv1_kernels_N256"] = k
    # ---- one rank's share of the 8-GPU step (local batch 1024, n_global 8192), graph replay
    n = GLOBAL_BATCH // 8
    xs = [torch.from_numpy(synth.mnist_like(n, seed=(1105, i))).cuda() for i in range(4)]
    ys = [torch.from_numpy(synth.labels(n, seed=(1106, i))).cuda() for i in range(4)]
    net = S.LeNet(n, math="tf32")
    p = prm.clone()
    g = torch.empty_like(p)
    med, mn = time_graph(lambda: net.step(p, g, xs[0], ys[0], GLOBAL_BATCH, lr=0.01), reps, flush)
    out["per_rank_step_local1024"] = {"us_per_step": round(1e3 * med, 2), "min_us": round(1e3 * mn, 2),
                                      "note": "one rank's compute at N = 8 (no allreduce: 1 GPU); "
                                              "8-GPU efficiency = t(8192) / (8 (t(1024) + t_allreduce))"}
    del net
    out["lenet512_step_N8192"] = lenet512_leg(S, peaks, flush, reps)
    return out


def lenet512_leg(S, peaks, flush, reps):
    """NEXT-4: the LeNet-512 step (affine 3136->512 + relu + dropout 0.5 + affine 512->10) at
    batch 8192, TF32, graph replay, with its per-stage breakdown (untimed eager pass)."""
    import torch
    import synth
    n = GLOBAL_BATCH
    xs = [torch.from_numpy(synth.mnist_like(n, seed=(1107, i))).cuda() for i in range(2)]
    ys = [torch.from_numpy(synth.labels(n, seed=(1108, i))).cuda() for i in range(2)]
    prm = torch.from_numpy(synth.lenet512_params(seed=(7,))).cuda()
    net = S.LeNet(n, math="tf32", model="lenet512", keep_p=0.5, seed=180204647)
    g = torch.empty_like(prm)
    med, mn = time_graph(lambda: net.step(prm, g, xs[0], ys[0], n, lr=0.01), reps, flush)
    # hidden-layer FLOPs: 3 GEMMs of 2 * n * 3136 * 512
    gemm_flop = 3 * 2.0 * n * 3136 * 512
    net.set_timing(True)
    for _ in range(3):
        net.step(prm, g, xs[1], ys[1], n, lr=0.01)
    torch.cuda.synchronize()
    stages = {k: round(v[0] / max(1, v[1]), 4) for k, v in net.get_timing(reset=True).items() if v[1]}
    net.set_timing(False)
    return {"N": n, "us_per_step": round(1e3 * med, 2), "min_us": round(1e3 * mn, 2),
            "images_per_s": round(n / (med * 1e-3), 1), "launch": "cuda_graph", "keep_p": 0.5,
            "params": int(net.num_params), "stage_avg_ms": stages,
            "hidden_gemm_flop_per_step": gemm_flop,
            "note": "F3h = hidden GEMM + bias/relu/dropout epilogue; B3h = dz3, dW3 (transpose + TMA GEMM), da2 GEMM"}


def oracle_per_config():
    """The fp64 oracle timed on each BASELINE config (bounded samples, scaled), host cores."""
    import oracle
    import synth
    res = {"cores": int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1)), "cpu_model": cpu_model()}

    def t(fn):
        t0 = time.perf_counter(); fn(); return time.perf_counter() - t0
    x = synth.mnist_like(8, seed=(1,)).astype(np.float64)
    f = synth.normal((32, 25), 0.3, seed=(2,)).astype(np.float64)
    dy = synth.normal((8, 32 * 784), seed=(3,)).astype(np.float64)
    res["cfg1_conv1_N8_ms"] = {
        "fwd": round(1e3 * t(lambda: oracle.conv2d_fwd(x, f, 8, 1, 28, 28, 32, 5, 5, (1, 1), (2, 2))), 2),
        "bwd_filter": round(1e3 * t(lambda: oracle.conv2d_bwd_filter(x, dy, 8, 1, 28, 28, 32, 5, 5, (1, 1), (2, 2))), 2),
        "bwd_data": round(1e3 * t(lambda: oracle.conv2d_bwd_data(f, dy, 8, 1, 28, 28, 32, 5, 5, (1, 1), (2, 2))), 2)}
    prm = synth.lenet_params(seed=(6,)).astype(np.float64)
    for name, n in (("cfg2_lenet_step_N64_s", 64), ("cfg3_lenet_step_N256_s", 256)):
        xx = synth.mnist_like(n, seed=(4, n)); yy = synth.labels(n, seed=(5, n))
        res[name] = round(t(lambda: oracle.sgd_update(prm, oracle.lenet_fwd_bwd(xx, yy, prm)[0], 0.01)), 3)
    c4 = {}
    for lname, (C, H, K, R, pd) in {"resnet3x3_C256_K256_14x14": (256, 14, 256, 3, 1),
                                   "resnet1x1_C1024_K256_14x14": (1024, 14, 256, 1, 0)}.items():
        ns = 2  # sample of the N = 128 layer, scaled x64
        xx, ff, bb, dd = synth.conv_problem_U(ns, C, H, H, K, R, R, H, H, seed=(7,))
        c4[lname] = {op: round(128 / ns * t(fn), 2) for op, fn in (
            ("fwd", lambda: oracle.conv2d_fwd(xx, ff, ns, C, H, H, K, R, R, (1, 1), (pd, pd), bias=bb)),
            ("bwd_filter", lambda: oracle.conv2d_bwd_filter(xx, dd, ns, C, H, H, K, R, R, (1, 1), (pd, pd))),
            ("bwd_data", lambda: oracle.conv2d_bwd_data(ff, dd, ns, C, H, H, K, R, R, (1, 1), (pd, pd))))}
    res["cfg4_layers_N128_s"] = c4
    res["cfg4_note"] = "N = 2 sample scaled x64 to N = 128"
    return res


def layer_section(S, peaks, quick=False):
    """conv2d GFLOP/s vs TF32 peak on the BJ ResNet-style layers (cfg 4) and the CSR
    conv1 bandwidth case (cfg 3), each op timed alone with an L2 flush between reps."""
    import torch
    import synth
    tf32_peak = peaks["tf32"]  # burst: each op is timed alone (bf16 measured x 1.125/2.25)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")  # 256 MB > L2
    out = {}
    reps = 5 if quick else 20
    for name, (N, C, H, W, K, R, S_, st, pd) in {
        "resnet3x3_C256_K256_14x14_N128": (128, 256, 14, 14, 256, 3, 3, 1, 1),
        "resnet1x1_C1024_K256_14x14_N128": (128, 1024, 14, 14, 256, 1, 1, 1, 0),
        "lenet_conv2_C32_K64_14x14_N8192": (8192, 32, 14, 14, 64, 5, 5, 1, 2),
        # ResNet-50 strided convs (NEXT-2, phase split onto the stride-1 tcgen05 kernels)
        "resnet50_stem7x7s2_C3_K64_224_N128": (128, 3, 224, 224, 64, 7, 7, 2, 3),
        "resnet50_3x3s2_C128_K128_56_N128": (128, 128, 56, 56, 128, 3, 3, 2, 1),
    }.items():
        P = (H + 2 * pd - R) // st + 1
        Q = (W + 2 * pd - S_) // st + 1
        x, f, b, dy = synth.conv_problem_U(N, C, H, W, K, R, S_, P, Q, seed=(1000,))
        x, f, b, dy = (torch.from_numpy(t).cuda() for t in (x, f, b, dy))
        d = S.conv_desc(N, C, H, W, K, R, S_, st, pd, "tf32")
        y = torch.empty(N, K * P * Q, device="cuda")
        dx = torch.empty(N, C * H * W, device="cuda")
        df = torch.empty(K, C * R * S_, device="cuda"); db = torch.empty(K, device="cuda")
        ws = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
        flops = 2.0 * N * K * C * R * S_ * P * Q
        res = {}
        for op, fn, nbytes in (
            ("fwd", lambda: S.sysml_conv2d(x, f, d, bias=b, out=y, workspace=ws), 4 * (x.numel() + f.numel() + K + y.numel())),
            ("bwd_filter", lambda: S.sysml_conv2d_bwd_filter(x, dy, d, df=df, db=db, workspace=ws), 4 * (x.numel() + dy.numel() + df.numel() + K)),
            ("bwd_data", lambda: S.sysml_conv2d_bwd_data(f, dy, d, dx=dx, workspace=ws), 4 * (f.numel() + dy.numel() + dx.numel())),
        ):
            med, mn = time_op(fn, reps, flush)
            tfs = flops / (med * 1e-3) / 1e12
            gbs = nbytes / (med * 1e-3) / 1e9
            res[op] = {"ms": round(med, 4), "tflops": round(tfs, 2), "frac_tf32_peak": round(tfs / tf32_peak, 4),
                       "gbs": round(gbs, 1), "frac_hbm": round(gbs / peaks["hbm"], 4),
                       "route": S.sysml_last_route()}
            if peaks.get("tf32_cublas"):
                res[op]["frac_tf32_cublas"] = round(tfs / peaks["tf32_cublas"], 4)
        out[name] = res
        del x, f, b, dy, y, dx
    # CSR conv1 (BJ cfg 3 shape, N = 16384 as the bandwidth headline)
    N = 2048 if quick else 16384
    xd = synth.mnist_like(N, seed=(1001,))
    rp, ci, v = synth.to_csr(xd)
    m = S.CSR(torch.from_numpy(rp).cuda(), torch.from_numpy(ci).cuda(), torch.from_numpy(v).cuda(), N, 784)
    f = torch.from_numpy(synth.normal((32, 25), 0.28, seed=(1002,))).cuda()
    b = torch.zeros(32, device="cuda")
    d = S.conv_desc(N, 1, 28, 28, 32, 5, 5, 1, 2, "tf32")
    y = torch.empty(N, 32 * 784, device="cuda")
    dy = torch.from_numpy(synth.normal((N, 32 * 784), seed=(1003,))).cuda()
    df = torch.empty(32, 25, device="cuda"); db = torch.empty(32, device="cuda")
    ws = torch.empty(1 << 26, dtype=torch.uint8, device="cuda")
    nnz = ci.size
    fwd_bytes = 4 * (N + 1) + 8 * nnz + 4 * (800 + 32) + 4 * N * 32 * 784
    bwf_bytes = 4 * (N + 1) + 8 * nnz + 4 * N * 32 * 784 + 4 * 832
    res = {"nnz": int(nnz), "density": round(nnz / (N * 784), 4)}
    pd = S.pool_desc(N, 32, 28, 28, 2, 2, 2, 0, True)
    pout = torch.empty(N, 32 * 196, device="cuda")
    parg = torch.empty(N, 32 * 196, dtype=torch.int32, device="cuda")
    fused_bytes = 4 * (N + 1) + 8 * nnz + 4 * (800 + 32) + 8 * N * 32 * 196
    for op, fn, nbytes in (("fwd", lambda: S.sysml_conv2d(m, f, d, bias=b, out=y, workspace=ws), fwd_bytes),
                           ("fwd_bias_relu_pool", lambda: S.sysml_conv2d_bias_relu_maxpool(
                               m, f, b, d, pd, out=pout, argmax=parg, workspace=ws), fused_bytes),
                           ("bwd_filter", lambda: S.sysml_conv2d_bwd_filter(m, dy, d, df=df, db=db, workspace=ws), bwf_bytes)):
        med, mn = time_op(fn, reps, flush)
        gbs = nbytes / (med * 1e-3) / 1e9
        res[op] = {"ms": round(med, 4), "gbs": round(gbs, 1), "frac_hbm": round(gbs / peaks["hbm"], 4),
                   "route": S.sysml_last_route()}
    out[f"csr_lenet_conv1_N{N}"] = res
    out["horizontal_fusion"] = horizontal_section(S, flush, reps)
    out["peak_note"] = ("frac_tf32_peak: of the burst TF32 denominator (measured bf16 x 0.5 = %.1f TFLOP/s); "
                        "frac_tf32_cublas: of cuBLAS TF32 measured live; frac_hbm: of measured HBM copy %.1f GB/s"
                        % (tf32_peak, peaks["hbm"]))
    return out


def horizontal_section(S, flush, reps):
    """NEXT-2 horizontal fusion: the ResNet bottleneck's conv1 and projection
    shortcut over one input, as two separate convs vs one call over the stacked bank."""
    import torch
    import synth
    out = {}
    for name, (N, C, H, W, ks, st) in {
        "resnet50_stage1_block1_conv1_64+proj_256_56x56_N128": (128, 64, 56, 56, (64, 256), 1),
        "resnet50v1_stage2_block1_conv1_128+proj_512_s2_56x56_N128": (128, 256, 56, 56, (128, 512), 2),
    }.items():
        P = (H - 1) // st + 1
        K = sum(ks)
        x = torch.from_numpy(synth.conv_problem_U(N, C, H, W, 1, 1, 1, P, P, seed=(1010,))[0]).cuda()
        fs = [torch.from_numpy(synth.normal((k, C), (2.0 / C) ** 0.5, seed=(1011, k))).cuda() for k in ks]
        dys = [torch.from_numpy(synth.normal((N, k * P * P), seed=(1012, k))).cuda() for k in ks]
        dy_cat = torch.cat([dy.view(N, k, -1) for dy, k in zip(dys, ks)], 1).view(N, -1).contiguous()
        ds = [S.conv_desc(N, C, H, W, k, 1, 1, st, 0, "tf32") for k in ks]
        d = S.conv_desc(N, C, H, W, K, 1, 1, st, 0, "tf32")
        ws = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
        ys = [torch.empty(N, k * P * P, device="cuda") for k in ks]
        y_cat = torch.empty(N, K * P * P, device="cuda")
        dx = torch.empty(N, C * H * W, device="cuda")
        dfs = [torch.empty(k, C, device="cuda") for k in ks]
        res = {"x_MB": round(4 * x.numel() / 1e6, 1)}
        sep = {
            "fwd": lambda: [S.sysml_conv2d(x, f, dd, out=y, workspace=ws) for f, dd, y in zip(fs, ds, ys)],
            "bwd_data": lambda: [S.sysml_conv2d_bwd_data(f, dy, dd, dx=dx, workspace=ws) for f, dy, dd in zip(fs, dys, ds)],
            "bwd_filter": lambda: [S.sysml_conv2d_bwd_filter(x, dy, dd, df=df, workspace=ws)
                                   for dy, dd, df in zip(dys, ds, dfs)],
        }
        fus = {
            "fwd": lambda: S.sysml_conv2d_multi(x, fs, d, out=y_cat, workspace=ws),
            "bwd_data": lambda: S.sysml_conv2d_multi_bwd_data(fs, dy_cat, d, dx=dx, workspace=ws),
            "bwd_filter": lambda: S.sysml_conv2d_multi_bwd_filter(x, dy_cat, d, ks, want_db=False, workspace=ws),
        }
        for op in ("fwd", "bwd_data", "bwd_filter"):
            ms_sep, _ = time_op(sep[op], reps, flush)
            ms_fus, _ = time_op(fus[op], reps, flush)
            res[op] = {"separate_ms": round(ms_sep, 4), "fused_ms": round(ms_fus, 4),
                       "speedup": round(ms_sep / ms_fus, 3), "route": S.sysml_last_route()}
        res["note"] = ("separate bwd_data = the two adjoints alone (their sum, which the fused call "
                       "returns, is not included)")
        out[name] = res
    return out


def ours_arm(args, world, rank, local):
    import torch
    import torch.distributed as dist
    import synth
    import paper_1802_04647_b200 as S

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    S.lib(build_if_missing=True)
    peaks = load_peaks()
    b = GLOBAL_BATCH // world
    math = args.math
    # data: ROTATE distinct input batches per rank, resident in HBM
    xs_host = [synth.mnist_like(b, seed=(rank, i)) for i in range(ROTATE)]
    ys_host = [synth.labels(b, seed=(100 + rank, i)) for i in range(ROTATE)]
    xs = [torch.from_numpy(x).cuda() for x in xs_host]
    ys = [torch.from_numpy(y).cuda() for y in ys_host]
    params = torch.from_numpy(synth.lenet_params(seed=(6,))).cuda()
    grads = torch.empty_like(params)
    loss = torch.empty(1, device="cuda")
    from paper_1802_04647_b200.dp import DataParallelLeNet
    dp = DataParallelLeNet(GLOBAL_BATCH, math=math)  # rank r: rows [r*b, (r+1)*b)
    net, comm = dp.net, dp.comm
    st = torch.cuda.current_stream()

    def step(i):
        dp.step(params, grads, xs[i % ROTATE], ys[i % ROTATE], lr=0.01, loss_sum=loss)

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    # the whole step (all kernels, the in-library NCCL allreduce and the SGD update) is
    # captured once per rotating input batch into a CUDA graph; the timed loop replays them
    graphs, graph_note = None, "eager"
    launches_per_step = None
    if not args.no_graph:
        try:
            cs = torch.cuda.Stream()
            cs.wait_stream(st)
            l_cap = S.sysml_launch_counter()
            graphs = []
            for r in range(ROTATE):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=cs):
                    dp.step(params, grads, xs[r], ys[r], lr=0.01, loss_sum=loss)
                graphs.append(g)
            launches_per_step = (S.sysml_launch_counter() - l_cap) / ROTATE
            st.wait_stream(cs)
            for i in range(2):
                graphs[i % ROTATE].replay()
            torch.cuda.synchronize()
            graph_note = "cuda_graph"
        except Exception as ex:  # fall back to eager launches
            graphs, graph_note = None, f"eager (graph capture failed: {type(ex).__name__})"
            torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.3)
    l0 = S.sysml_launch_counter()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for i in range(args.steps):
        if graphs is not None:
            graphs[i % ROTATE].replay()
        else:
            step(i)
    e1.record(st)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = S.sysml_launch_counter() - l0
    if graphs is not None:  # graph nodes: the library's kernels of one captured step
        launches = int(round(launches_per_step * args.steps))
    clocks = clk.stop()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    # per-stage breakdown from an untimed eager pass with the library's stage events
    net.set_timing(True)
    net.get_timing(reset=True)
    for i in range(args.steps):
        step(i)
    torch.cuda.synchronize()
    net.set_timing(False)
    stages = net.get_timing()
    value = GLOBAL_BATCH * args.steps / (ms * 1e-3)

    # ---- end to end through the host-input C-ABI entry point (pinned host batches)
    xs_pin = [torch.from_numpy(x).pin_memory() for x in xs_host]
    ys_pin = [torch.from_numpy(y).pin_memory() for y in ys_host]
    # pipelined host loop: step i computes while batch i+1 is copied host -> device (one batch
    # H2D and one loss D2H per step inside the timed region; the warm-up prefetches batch 0)
    def host_step(i):
        net.step_host_pipelined(params, grads, xs_pin[i % ROTATE], ys_pin[i % ROTATE], GLOBAL_BATCH,
                                next_x=xs_pin[(i + 1) % ROTATE], next_labels=ys_pin[(i + 1) % ROTATE],
                                nccl_comm=comm)
    for i in range(-2, 0):
        host_step(i)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e2 = torch.cuda.Event(enable_timing=True); e3 = torch.cuda.Event(enable_timing=True)
    e2.record(st)
    for i in range(args.steps):
        host_step(i)
    e3.record(st)
    torch.cuda.synchronize()
    ms_e2e = e2.elapsed_time(e3)
    if world > 1:
        t = torch.tensor([ms_e2e], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_e2e = float(t.item())
    e2e_value = GLOBAL_BATCH * args.steps / (ms_e2e * 1e-3)

    # ---- scoring (P:193-202 parfor-style row-partitioned scoring): forward + softmax/argmax of
    # the local rows through sysml_lenet_predict; replicas, no collective
    for i in range(3):
        net.predict(params, xs[i % ROTATE])
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e4 = torch.cuda.Event(enable_timing=True); e5 = torch.cuda.Event(enable_timing=True)
    e4.record(st)
    for i in range(args.steps):
        net.predict(params, xs[i % ROTATE])
    e5.record(st)
    torch.cuda.synchronize()
    ms_score = e4.elapsed_time(e5)
    if world > 1:
        t = torch.tensor([ms_score], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_score = float(t.item())
    score_value = GLOBAL_BATCH * args.steps / (ms_score * 1e-3)

    # ---- roofline of the dominant stage.  One denominator for the whole line: the burst peak
    # for a timed region that ran at full clocks (this ~40 ms step loop), the sustained one
    # when the clock record shows the power-capped regime.
    reg = regime(clocks, peaks["sm_max"])
    tf32_pk = peaks["tf32"] if reg == "burst" else peaks["tf32_sus"]
    stage_rows = {}
    for name, (tot_ms, calls) in stages.items():
        if calls == 0:
            continue
        fl, by, bound = STAGE_WORK[name]
        avg = tot_ms / calls
        tfl = fl * b / (avg * 1e-3) / 1e12
        gbs = by * b / (avg * 1e-3) / 1e9
        row = {"avg_ms": round(avg, 4), "share": round(tot_ms / max(ms, 1e-9), 4),
               "tflops": round(tfl, 2), "gbs": round(gbs, 1), "bound": bound}
        if bound == "tensor" and math == "tf32":
            row["frac"] = round(tfl / tf32_pk, 4)
        elif bound == "tensor":
            row["bound"] = "alu"
            row["frac"] = round(tfl / peaks["fp32_alu"], 4)
        else:
            row["frac"] = round(gbs / peaks["hbm"], 4)
        stage_rows[name] = row
    dom = max(stage_rows, key=lambda k: stage_rows[k]["avg_ms"])
    fl, by, bound = STAGE_WORK[dom]
    avg_s = stage_rows[dom]["avg_ms"] * 1e-3
    if bound == "tensor" and math == "tf32":
        achieved = fl * b / avg_s / 1e12
        roof = {"bound": "tensor", "achieved": round(achieved, 2), "peak": round(tf32_pk, 1), "unit": "TFLOP/s",
                "frac": round(achieved / tf32_pk, 4),
                "peak_note": f"TF32 {reg} = measured bf16 {reg} x 0.5 (nominal 1.125/2.25 PF); regime from the clock record"}
        if peaks.get("tf32_cublas"):
            roof["frac_tf32_cublas"] = round(achieved / peaks["tf32_cublas"], 4)
        roof["frac_tf32_spec"] = round(achieved / TF32_SPEC_TFLOPS, 4)
    elif bound == "tensor":
        achieved = fl * b / avg_s / 1e12
        roof = {"bound": "alu", "achieved": round(achieved, 2), "peak": round(peaks["fp32_alu"], 1), "unit": "TFLOP/s",
                "frac": round(achieved / peaks["fp32_alu"], 4), "peak_note": "148 SM x 128 FFMA x 2 x sm_max_mhz"}
    else:
        achieved = by * b / avg_s / 1e9
        roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peaks["hbm"], "unit": "GB/s",
                "frac": round(achieved / peaks["hbm"], 4)}
    traffic = None
    try:  # DRAM bytes of the dominant kernel from one ncu --set full capture (profiles/)
        t = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json"))).get(dom)
        if t:
            traffic = round(t["dram_bytes_per_image"] * b)
    except (OSError, ValueError):
        pass
    roof.update({"kernel": dom, "traffic": traffic, "algorithmic_bytes": by * b, "algorithmic_flops": fl * b,
                 "regime": reg, "peak_src": peaks["src"]})

    result = {
        "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 4), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "tf32" if math == "tf32" else "f32", "data": "synthetic",
        "config": {"workload": "DP LeNet minibatch SGD (BJ configs[4]): conv5x5(32)+relu+pool2 -> conv5x5(64)+relu+pool2 "
                               "-> affine(3136->10) -> softmax-CE, SGD lr 0.01",
                   "global_batch": GLOBAL_BATCH, "local_batch": b, "input": "dense MNIST-shaped (density ~0.19)",
                   "parallelism": f"dp{world}", "l2": f"{ROTATE} rotating input batches + ~0.6 GB/step activations >> 126 MB L2",
                   "launch": graph_note},
        "scoring": {"value": round(score_value, 1), "unit": UNIT,
                    "mode": "sysml_lenet_predict: forward + softmax / argmax of the local rows, row-partitioned replicas (no collective), device-resident batches"},
        "e2e": {"value": round(e2e_value, 1), "unit": UNIT, "h2d_bytes_per_step": b * 784 * 4 + b * 4,
                "d2h_bytes_per_step": 4, "mode": "sysml_lenet_step_host_pipelined: pinned host batches, batch i+1 copied H2D while step i computes, loss read back every step"},
        "gpu_launches": int(launches),
        "allreduce": ("in-library ncclAllReduce (torch ProcessGroupNCCL communicator)" if dp.use_lib_nccl
                      else ("torch.distributed.all_reduce" if world > 1 else "none (1 GPU)")),
        "clocks": clocks,
        "roofline": roof,
        "stages": stage_rows,
    }
    if rank == 0 and world == 1 and not args.no_layers:
        try:
            peaks["tf32_cublas"] = tf32_cublas_peak()
        except Exception as ex:  # the measuring stick is optional; the bf16-derived peak stays
            peaks["tf32_cublas"] = None
            result["tf32_cublas_error"] = f"{type(ex).__name__}: {ex}"
        result["peaks"] = {"hbm_gbs": peaks["hbm"], "tf32_burst_tflops": round(peaks["tf32"], 1),
                           "tf32_sustained_tflops": round(peaks["tf32_sus"], 1),
                           "tf32_cublas_measured_tflops": peaks["tf32_cublas"],
                           "tf32_spec_tflops": TF32_SPEC_TFLOPS, "fp32_alu_tflops": round(peaks["fp32_alu"], 1),
                           "src": peaks["src"]}
        if peaks["tf32_cublas"]:
            result["roofline"]["frac_tf32_cublas"] = (round(result["roofline"]["achieved"] / peaks["tf32_cublas"], 4)
                                                      if result["roofline"]["bound"] == "tensor" else None)
        result["layers"] = layer_section(S, peaks, quick=args.quick)
        try:
            for leg_name, leg in config_legs(S, peaks, quick=args.quick).items():
                result[leg_name] = leg
        except Exception as ex:  # keep the headline line even if a side leg fails
            result["config_legs_error"] = f"{type(ex).__name__}: {ex}"
    if rank == 0 and world == 1 and not args.no_cpu:
        v, n, t, cores = cpu_oracle_rate()
        result["cpu_baseline"] = {"value": round(v, 3), "unit": UNIT, "cores": cores, "kind": "oracle",
                                  "cpu_model": cpu_model(),
                                  "sample": f"fp64 oracle LeNet fwd+bwd+SGD on {n} images ({t:.1f} s)"}
        result["oracle_per_config"] = oracle_per_config()
    if rank == 0:
        print(json.dumps(result), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--math", default="tf32", choices=["tf32", "fp32"])
    ap.add_argument("--no-layers", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="launch the step eagerly instead of replaying CUDA graphs")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        spawn_ranks(args.gpus)  # does not return
    world, rank, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world} ranks were launched")
    if args.impl == "reference":
        reference_arm(args, world, rank)
        return
    ours_arm(args, world, rank, local)


if __name__ == "__main__":
    main()
