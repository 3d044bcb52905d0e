"""GPU parity of horizontal fusion for shared inputs (NEXT-2): several convs over
ONE input run as one conv over the stacked filter bank.  Each op's result is compared with
the fp64 oracle run on that op ALONE (fwd, bwd_filter) and bwd_data with the sum of the
oracle's per-op adjoints -- the fusion must change nothing but the schedule."""
import numpy as np
import pytest
import torch

import oracle
import synth

from tests.test_gpu_parity import TOL, S, assert_close, dev, host  # noqa: F401

pytestmark = pytest.mark.gpu

# N, C, H, W, R, S, stride, pad, k_counts
CASES = [
    (3, 64, 9, 9, 1, 1, 1, 0, (16, 48)),            # bottleneck conv1 + projection (stride 1)
    (2, 32, 14, 14, 1, 1, 2, 0, (32, 64)),          # ResNet v1 first block: both 1x1/2
    (2, 32, 10, 10, 3, 3, 1, 1, (24, 40, 8)),       # three 3x3 branches over one map
    (4, 1, 28, 28, 5, 5, 1, 2, (16, 16)),           # C = 1 (KS operand mode), two banks
    (2, 16, 11, 7, 3, 3, 2, 1, (5, 11)),            # strided 3x3, ragged widths
]


@pytest.mark.parametrize("math", ["fp32", "tf32"])
@pytest.mark.parametrize("case", CASES)
def test_horizontal_fusion_vs_oracle_per_op(S, math, case):
    N, C, H, W, R, S_, st, pd, ks = case
    P = oracle.out_extent(H, pd, R, st)
    Q = oracle.out_extent(W, pd, S_, st)
    K = sum(ks)
    x, _, _, _ = synth.conv_problem_U(N, C, H, W, 1, R, S_, P, Q, seed=(790, C))
    fs, bs, dys = [], [], []
    for i, k in enumerate(ks):
        _, f, b, dy = synth.conv_problem_U(N, C, H, W, k, R, S_, P, Q, seed=(791, i, C))
        fs.append(f); bs.append(b); dys.append(dy)
    d = S.conv_desc(N, C, H, W, K, R, S_, st, pd, math)
    # dy_cat: op i's channels are the slice [k_0 + ... + k_{i-1}, ...) of each row
    dy_cat = np.concatenate([dy.reshape(N, k, P * Q) for dy, k in zip(dys, ks)], axis=1).reshape(N, -1)
    y = host(S.sysml_conv2d_multi(dev(x), [dev(f) for f in fs], d, biases=[dev(b) for b in bs]))
    y = y.reshape(N, K, P * Q)
    dx = host(S.sysml_conv2d_multi_bwd_data([dev(f) for f in fs], dev(dy_cat), d))
    dfs, dbs = S.sysml_conv2d_multi_bwd_filter(dev(x), dev(dy_cat), d, ks)
    k0 = 0
    dx_ref = np.zeros((N, C * H * W))
    for i, k in enumerate(ks):
        ref = oracle.conv2d_fwd(x, fs[i], N, C, H, W, k, R, S_, (st, st), (pd, pd), bias=bs[i])
        assert_close(y[:, k0:k0 + k].reshape(N, -1), ref, TOL[math], f"fwd op {i}")
        dfr, dbr = oracle.conv2d_bwd_filter(x, dys[i], N, C, H, W, k, R, S_, (st, st), (pd, pd))
        assert_close(host(dfs[i]), dfr, TOL[math], f"df op {i}")
        assert_close(host(dbs[i]), dbr, TOL[math], f"db op {i}")
        dx_ref += oracle.conv2d_bwd_data(fs[i], dys[i], N, C, H, W, k, R, S_, (st, st), (pd, pd))
        k0 += k
    assert_close(dx, dx_ref, TOL[math], "dx = sum of the ops' adjoints")
    assert "horizontal fusion" in S.sysml_last_route()


def test_horizontal_fusion_csr_input_and_errors(S):
    N = 6
    x = synth.mnist_like(N, seed=(795,))
    rp, ci, v = synth.to_csr(x)
    m = S.CSR(dev(rp, torch.int32), dev(ci, torch.int32), dev(v), N, 784)
    ks = (8, 24)
    fs = [synth.conv_problem_U(N, 1, 28, 28, k, 5, 5, 28, 28, seed=(796, k))[1] for k in ks]
    d = S.conv_desc(N, 1, 28, 28, 32, 5, 5, 1, 2, "tf32")
    y = host(S.sysml_conv2d_multi(m, [dev(f) for f in fs], d)).reshape(N, 32, 784)
    for i, (k0, k) in enumerate(((0, 8), (8, 24))):
        ref = oracle.conv2d_fwd(x, fs[i], N, 1, 28, 28, k, 5, 5, (1, 1), (2, 2))
        assert_close(y[:, k0:k0 + k].reshape(N, -1), ref, TOL["tf32"], f"csr op {i}")
    bad = S.conv_desc(N, 1, 28, 28, 31, 5, 5, 1, 2, "tf32")   # K != sum(k_counts)
    with pytest.raises(S.SysmlError, match="sum of k_counts"):
        S.sysml_conv2d_multi(m, [dev(f) for f in fs], bad)
