"""GPU parity: the CUDA path (through the C ABI) vs the fp64 oracle, element by element,
on identical seeded inputs (synth/).  Tolerances (BJ north_star):
  fp32 CUDA-core kernels  max|gpu - ref| <= 1e-4 * max|ref|
  TF32 tensor-core kernels max|gpu - ref| <= 5e-3 * max|ref|
  pooling argmax / index outputs: bit-exact.
"""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

TOL = {"fp32": 1e-4, "tf32": 5e-3}


@pytest.fixture(scope="module")
def S():
    assert torch.cuda.is_available(), "GPU tests need CUDA"
    import paper_1802_04647_b200 as s
    s.lib()
    return s


def dev(a, dtype=torch.float32):
    return torch.from_numpy(np.ascontiguousarray(a)).to(device="cuda", dtype=dtype)


def host(t):
    return t.detach().cpu().numpy()


def assert_close(gpu, ref, tol, what=""):
    gpu = np.asarray(gpu, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert gpu.shape == ref.shape, (gpu.shape, ref.shape)
    scale = max(np.abs(ref).max(initial=0.0), 1e-30)
    err = np.abs(gpu - ref).max(initial=0.0)
    assert err <= tol * scale, f"{what}: max|err| {err:.3e} > {tol:g} * max|ref| {scale:.3e}"


def assert_valid_argmax(arg, z, oref, tol, what="", exact_ref=None):
    """SURVEY §8(c) protocol 2 (fused conv+bias+relu+pool on continuous data): every GPU index
    lies inside its own pooling window and the oracle's relu(z) at that index is within
    tolerance of the oracle's window max.  Returns the number of argmax flips against the
    oracle's first-occurrence index (reported, not gated; exact_ref, when given, gates them
    to zero)."""
    a = np.asarray(arg).astype(np.int64)
    zr = np.maximum(np.asarray(z, np.float64), 0.0)
    assert a.min(initial=0) >= 0 and a.max(initial=0) < zr.shape[1], f"{what}: argmax out of the row"
    picked = np.take_along_axis(zr, a, axis=1)
    scale = max(np.abs(oref).max(initial=0.0), 1e-30)
    err = np.abs(picked - oref).max(initial=0.0)
    assert err <= tol * scale, f"{what}: relu(z) at the GPU argmax is {err:.3e} off the window max"
    flips = int((a != exact_ref).sum()) if exact_ref is not None else 0
    return flips


def assert_argmax_in_window(arg, C, H, W, P, Q, R, S_, stride):
    """Each argmax (c*H + h)*W + w of pooled output (c, p, q) lies in that output's window."""
    a = np.asarray(arg).astype(np.int64).reshape(arg.shape[0], C, P, Q)
    c = a // (H * W); h = (a // W) % H; w = a % W
    cc, pp, qq = np.meshgrid(np.arange(C), np.arange(P), np.arange(Q), indexing="ij")
    assert np.all(c == cc[None])
    assert np.all((h >= pp[None] * stride[0]) & (h < pp[None] * stride[0] + R))
    assert np.all((w >= qq[None] * stride[1]) & (w < qq[None] * stride[1] + S_))


# N, C, H, W, K, R, S, stride, pad  -- several tiles + ragged tails, plus the BJ layer shapes
CONV_SHAPES = [
    (8, 1, 28, 28, 32, 5, 5, 1, 2),      # BJ cfg 1: LeNet conv1
    (5, 32, 14, 14, 64, 5, 5, 1, 2),     # LeNet conv2
    (3, 5, 11, 9, 7, 3, 3, 2, 1),        # ragged, stride 2
    (2, 3, 10, 13, 70, 3, 2, 1, (1, 0)), # K > 64 tile, rectangular kernel
    (2, 256, 14, 14, 256, 3, 3, 1, 1),   # BJ cfg 4 (i) 3x3 C=K=256 at N=2
    (2, 1024, 14, 14, 256, 1, 1, 1, 0),  # BJ cfg 4 (ii) 1x1 1024->256 at N=2
    (1, 2, 5, 5, 3, 5, 5, 1, 0),         # P = Q = 1
    (3, 1, 17, 23, 20, 7, 3, 1, (3, 1)), # C = 1 (KS operand mode), tall kernel, ragged
    (2, 1, 9, 30, 5, 2, 8, 1, (0, 4)),   # C = 1, S = 8 (both K halves full)
    (2, 4, 9, 9, 1, 3, 3, 1, 1),         # K = 1 (bwd_data input has one channel)
    (3, 48, 6, 6, 40, 1, 1, 1, 0),       # 1x1 TMA wgrad: one 128-filter tile, 48-channel tile
    (2, 32, 4, 4, 300, 1, 1, 1, 0),      # 1x1 TMA wgrad: K > 256 (two filter-pair tiles), ragged
    (2, 16, 9, 11, 136, 3, 3, 1, 1),     # framed TMA wgrad: K > 128 (two filter tiles), 16-ch tile
    (2, 32, 10, 12, 48, 3, 3, 1, 0),     # framed TMA wgrad: pad 0, rectangular
    (4, 64, 14, 14, 96, 1, 1, 2, 0),     # 1x1 stride 2 (ResNet downsample): tcgen05 on the output grid
    (2, 24, 9, 11, 40, 1, 1, 2, 0),      # 1x1 stride 2, odd extents (floor)
    (2, 32, 16, 16, 48, 1, 1, 2, 0),     # 1x1 stride 2, P*Q % 4 == 0: strided TMA bwd_filter
    # strided R, S > 1 (TF32: phase split + stride-1 tcgen05 kernels, phase.cu)
    (2, 3, 32, 30, 64, 7, 7, 2, 3),      # ResNet-50 stem 7x7/2 pad 3, small image
    (2, 64, 15, 15, 64, 3, 3, 2, 1),     # 3x3/2 odd extent (floor drops the last row)
    (2, 128, 16, 16, 128, 3, 3, 2, 1),   # ResNet-50 stage-transition 3x3/2
    (2, 8, 11, 13, 24, 5, 3, 3, (2, 1)), # stride 3, rectangular kernel, asymmetric pad
    (2, 16, 12, 10, 32, 3, 3, (2, 1), 1),  # asymmetric stride
    (3, 12, 9, 9, 20, 2, 2, 2, 0),       # 2x2/2 (phase split has R' = S' = 1)
]


def _conv_case(shape, seed):
    N, C, H, W, K, R, S_, st, pd = shape
    pd = pd if isinstance(pd, tuple) else (pd, pd)
    st = st if isinstance(st, tuple) else (st, st)
    P = oracle.out_extent(H, pd[0], R, st[0])
    Q = oracle.out_extent(W, pd[1], S_, st[1])
    x, f, b, dy = synth.conv_problem_U(N, C, H, W, K, R, S_, P, Q, seed=(seed,))
    return (N, C, H, W, K, R, S_, st, pd, P, Q), x, f, b, dy


@pytest.mark.parametrize("math", ["fp32", "tf32"])
@pytest.mark.parametrize("shape", CONV_SHAPES)
def test_conv_fwd_bwd_parity(S, shape, math):
    (N, C, H, W, K, R, S_, st, pd, P, Q), x, f, b, dy = _conv_case(shape, 100)
    d = S.conv_desc(N, C, H, W, K, R, S_, st, pd, math)
    y = S.sysml_conv2d(dev(x), dev(f), d, bias=dev(b))
    yref = oracle.conv2d_fwd(x, f, N, C, H, W, K, R, S_, st, pd, bias=b)
    assert_close(host(y), yref, TOL[math], "fwd")
    y0 = S.sysml_conv2d(dev(x), dev(f), d)
    assert_close(host(y0), oracle.conv2d_fwd(x, f, N, C, H, W, K, R, S_, st, pd), TOL[math], "fwd nobias")
    df, db = S.sysml_conv2d_bwd_filter(dev(x), dev(dy), d)
    dfr, dbr = oracle.conv2d_bwd_filter(x, dy, N, C, H, W, K, R, S_, st, pd)
    assert_close(host(df), dfr, TOL[math], "bwd_filter")
    assert_close(host(db), dbr, 1e-4, "db")
    dx = S.sysml_conv2d_bwd_data(dev(f), dev(dy), d)
    assert_close(host(dx), oracle.conv2d_bwd_data(f, dy, N, C, H, W, K, R, S_, st, pd), TOL[math], "bwd_data")


@pytest.mark.parametrize("math", ["fp32", "tf32"])
def test_conv_dyadic_grid_exact(S, math):
    # family G: every partial sum is exact in fp32 and TF32 -> bit-exact vs fp64
    N, C, H, W, K, R, S_ = 2, 64, 14, 14, 64, 3, 3
    x, f, b, dy = synth.conv_problem_G(N, C, H, W, K, R, S_, 14, 14)
    d = S.conv_desc(N, C, H, W, K, R, S_, 1, 1, math)
    y = host(S.sysml_conv2d(dev(x), dev(f), d, bias=dev(b)))
    assert np.array_equal(y, oracle.conv2d_fwd(x, f, N, C, H, W, K, R, S_, (1, 1), (1, 1), bias=b))
    df, db = S.sysml_conv2d_bwd_filter(dev(x), dev(dy), d)
    dfr, dbr = oracle.conv2d_bwd_filter(x, dy, N, C, H, W, K, R, S_, (1, 1), (1, 1))
    assert np.array_equal(host(df), dfr) and np.array_equal(host(db), dbr)
    dx = host(S.sysml_conv2d_bwd_data(dev(f), dev(dy), d))
    assert np.array_equal(dx, oracle.conv2d_bwd_data(f, dy, N, C, H, W, K, R, S_, (1, 1), (1, 1)))


@pytest.mark.parametrize("math", ["fp32", "tf32"])
def test_conv_determinism(S, math):
    (N, C, H, W, K, R, S_, st, pd, P, Q), x, f, b, dy = _conv_case(CONV_SHAPES[1], 7)
    d = S.conv_desc(N, C, H, W, K, R, S_, st, pd, math)
    outs = []
    for _ in range(2):
        y = S.sysml_conv2d(dev(x), dev(f), d, bias=dev(b))
        df, db = S.sysml_conv2d_bwd_filter(dev(x), dev(dy), d)
        dx = S.sysml_conv2d_bwd_data(dev(f), dev(dy), d)
        outs.append([host(t).tobytes() for t in (y, df, db, dx)])
    assert outs[0] == outs[1]


POOL_CASES = [
    # N, C, H, W, R, S, stride, pad
    (4, 32, 28, 28, 2, 2, 2, 0),
    (3, 5, 7, 9, 3, 3, 2, 1),   # overlapping + padding
    (2, 3, 6, 7, 2, 3, (1, 2), (1, 1)),
    (2, 4, 7, 7, 2, 2, 2, 0),   # trailing row/col not covered
]


@pytest.mark.parametrize("relu", [True, False])
@pytest.mark.parametrize("case", POOL_CASES)
def test_relu_maxpool_and_bwd_bit_exact(S, case, relu):
    N, C, H, W, R, S_, st, pd = case
    st = st if isinstance(st, tuple) else (st, st)
    pd = pd if isinstance(pd, tuple) else (pd, pd)
    rng = synth.rng(200)
    for x in (synth.uniform((N, C * H * W), seed=(201,)),
              (rng.integers(-1, 2, size=(N, C * H * W)) / 2.0).astype(np.float32)):  # ties + zeros
        d = S.pool_desc(N, C, H, W, R, S_, st, pd, relu)
        out, arg = S.sysml_relu_maxpool(dev(x), d)
        oref, aref = oracle.relu_maxpool(x, N, C, H, W, R, S_, st, pd, relu=relu)
        assert np.array_equal(host(arg), aref)
        assert np.array_equal(host(out).astype(np.float64) + 0.0, oref + 0.0)  # +-0 canonicalised
        P, Q = d.P, d.Q
        dout = synth.normal((N, C * P * Q), seed=(202,))
        for mask in (None, out):
            dx = S.sysml_maxpool_bwd(arg, dev(dout), d, out_mask=mask)
            dxr = oracle.maxpool_bwd(aref, dout, N, C, H, W, P, Q,
                                     out_mask=None if mask is None else oref)
            if st[0] >= R and st[1] >= S_:
                assert np.array_equal(host(dx).astype(np.float64), dxr)  # one term per element
            else:
                assert_close(host(dx), dxr, 1e-6, "maxpool_bwd overlap")


def test_bias_add(S):
    y = synth.uniform((3, 7 * 30), seed=(300,))
    b = synth.uniform((7,), seed=(301,))
    t = dev(y)
    S.sysml_bias_add(t, dev(b), 3, 7, 30)
    assert_close(host(t), oracle.bias_add(y, b, 3, 7, 30), 1e-7, "bias_add")


@pytest.mark.parametrize("math", ["fp32", "tf32"])
def test_fused_conv_bias_relu_maxpool_dyadic_bit_exact(S, math):
    # LeNet conv2 block on the dyadic grid: conv exact -> argmax bit-exact (SURVEY §8(c) protocol 2)
    N = 6
    x = synth.dyadic((N, 32 * 14 * 14), 0, 4, 4, seed=(400,))
    f = synth.dyadic((64, 800), -3, 3, 64, seed=(401,))
    b = synth.dyadic((64,), -3, 3, 16, seed=(402,))
    cd = S.conv_desc(N, 32, 14, 14, 64, 5, 5, 1, 2, math)
    pd = S.pool_desc(N, 64, 14, 14, 2, 2, 2, 0, True)
    out, arg = S.sysml_conv2d_bias_relu_maxpool(dev(x), dev(f), dev(b), cd, pd)
    z = oracle.conv2d_fwd(x, f, N, 32, 14, 14, 64, 5, 5, (1, 1), (2, 2), bias=b)
    oref, aref = oracle.relu_maxpool(z, N, 64, 14, 14, 2, 2, (2, 2), (0, 0), relu=True)
    assert np.array_equal(host(arg), aref)
    assert np.array_equal(host(out).astype(np.float64), oref)


# (N, K, H, W, R, pad): C = 1 conv + pool with the 2x2 window in the MMA N dimension
# (conv1_pool.cu): LeNet conv1, a 3x3 kernel with K <= 16, a tall 7x7 kernel, ragged
# window count (N*Pp*Qp not a multiple of 256)
C1P_SHAPES = [(7, 32, 28, 28, 5, 2), (3, 12, 10, 14, 3, 0), (2, 20, 16, 12, 7, 2)]


@pytest.mark.parametrize("shape", C1P_SHAPES)
def test_conv1_pool_dyadic_bit_exact(S, shape):
    N, K, H, W, R, pd = shape
    x = synth.dyadic((N, H * W), 0, 4, 4, seed=(410,))
    x[x < 0.5] = 0.0  # zero-heavy: window ties at 0 exercise the first-occurrence rule
    f = synth.dyadic((K, R * R), -3, 3, 16, seed=(411,))
    b = synth.dyadic((K,), -3, 3, 16, seed=(412,))
    P = H + 2 * pd - R + 1
    Q = W + 2 * pd - R + 1
    cd = S.conv_desc(N, 1, H, W, K, R, R, 1, pd, "tf32")
    pdsc = S.pool_desc(N, K, P, Q, 2, 2, 2, 0, True)
    out, arg = S.sysml_conv2d_bias_relu_maxpool(dev(x), dev(f), dev(b), cd, pdsc)
    z = oracle.conv2d_fwd(x, f, N, 1, H, W, K, R, R, (1, 1), (pd, pd), bias=b)
    oref, aref = oracle.relu_maxpool(z, N, K, P, Q, 2, 2, (2, 2), (0, 0), relu=True)
    assert np.array_equal(host(arg), aref)
    assert np.array_equal(host(out).astype(np.float64), oref)


@pytest.mark.parametrize("math", ["fp32", "tf32"])
def test_fused_conv_pool_continuous_valid_argmax(S, math):
    N = 5
    x = synth.mnist_like(N, seed=(410,))
    f = synth.normal((32, 25), np.sqrt(2 / 25), seed=(411,))
    b = synth.normal((32,), 0.1, seed=(412,))
    cd = S.conv_desc(N, 1, 28, 28, 32, 5, 5, 1, 2, math)
    pd = S.pool_desc(N, 32, 28, 28, 2, 2, 2, 0, True)
    out, arg = S.sysml_conv2d_bias_relu_maxpool(dev(x), dev(f), dev(b), cd, pd)
    z = oracle.conv2d_fwd(x, f, N, 1, 28, 28, 32, 5, 5, (1, 1), (2, 2), bias=b)
    oref, aref = oracle.relu_maxpool(z, N, 32, 28, 28, 2, 2, (2, 2), (0, 0), relu=True)
    assert_close(host(out), oref, TOL[math], "pooled")
    # valid argmax: the oracle's relu(z) at the GPU index is within tolerance of the oracle max
    a = host(arg)
    assert_argmax_in_window(a, 32, 28, 28, 14, 14, 2, 2, (2, 2))
    flips = assert_valid_argmax(a, z, oref, TOL[math], "dense fused", exact_ref=aref)
    print(f"dense fused {math}: {flips} argmax flips of {a.size} windows (valid argmax holds)")


# ---------------------------------------------------------------------------- CSR

def _csr_dev(S, dense):
    rp, ci, v = synth.to_csr(dense)
    return S.CSR(dev(rp, torch.int32), dev(ci, torch.int32), dev(v), dense.shape[0], dense.shape[1]), (rp, ci, v)


@pytest.mark.parametrize("N", [12, 37])
@pytest.mark.parametrize("math", ["fp32", "tf32"])
def test_csr_conv_fwd_bwd_filter(S, math, N):
    x = synth.mnist_like(N, seed=(500,))
    x[0] = 0.0                                    # empty row
    x[1] = synth.uniform((784,), 0.01, 1.0, seed=(501,))  # fully dense row
    x[2, [0, 27, 28 * 27, 783]] = [0.5, 0.25, 0.75, 1.0]   # border non-zeros
    m, (rp, ci, v) = _csr_dev(S, x)
    assert S.sysml_csr_check(m) == 0
    xd = oracle.csr_densify(rp, ci, v, N, 784)
    f = synth.normal((32, 25), np.sqrt(2 / 25), seed=(502,))
    b = synth.normal((32,), 0.1, seed=(503,))
    dy = synth.normal((N, 32 * 784), seed=(504,))
    d = S.conv_desc(N, 1, 28, 28, 32, 5, 5, 1, 2, math)
    y = S.sysml_conv2d(m, dev(f), d, bias=dev(b))
    assert_close(host(y), oracle.conv2d_fwd(xd, f, N, 1, 28, 28, 32, 5, 5, (1, 1), (2, 2), bias=b), TOL[math], "csr fwd")
    df, db = S.sysml_conv2d_bwd_filter(m, dev(dy), d)
    dfr, dbr = oracle.conv2d_bwd_filter(xd, dy, N, 1, 28, 28, 32, 5, 5, (1, 1), (2, 2))
    assert_close(host(df), dfr, 1e-4, "csr bwd_filter")
    assert_close(host(db), dbr, 1e-4, "csr db")
    pd = S.pool_desc(N, 32, 28, 28, 2, 2, 2, 0, True)
    out, arg = S.sysml_conv2d_bias_relu_maxpool(m, dev(f), dev(b), d, pd)
    z = oracle.conv2d_fwd(xd, f, N, 1, 28, 28, 32, 5, 5, (1, 1), (2, 2), bias=b)
    oref, aref = oracle.relu_maxpool(z, N, 32, 28, 28, 2, 2, (2, 2), (0, 0))
    assert_close(host(out), oref, TOL[math], "csr fused")
    a = host(arg)
    assert_argmax_in_window(a, 32, 28, 28, 14, 14, 2, 2, (2, 2))
    flips = assert_valid_argmax(a, z, oref, TOL[math], "csr fused", exact_ref=aref)
    print(f"csr fused {math} N={N}: {flips} argmax flips of {a.size} windows (valid argmax holds)")


# (N, C, H, W, K, R, S, pad): the lane-per-filter K8 path (C=1, K<=32) and the fallback
CSR_WGRAD_SHAPES = [
    (5, 1, 12, 16, 20, 3, 3, 1),
    (3, 1, 12, 16, 7, 5, 5, 0),
    (4, 1, 9, 10, 32, 5, 5, 2),    # P*Q = 90: not a multiple of 4 -> fallback kernel
    (3, 2, 8, 8, 5, 3, 3, 1),      # C = 2 -> fallback kernel
]


@pytest.mark.parametrize("shape", CSR_WGRAD_SHAPES)
def test_csr_bwd_filter_shapes(S, shape):
    N, C, H, W, K, R, S_, pd = shape
    P, Q = H + 2 * pd - R + 1, W + 2 * pd - S_ + 1
    x = synth.uniform((N, C * H * W), 0.0, 1.0, seed=(520,))
    x[x < 0.7] = 0.0
    x[0, :] = 0.0
    m, (rp, ci, v) = _csr_dev(S, x)
    dy = synth.normal((N, K * P * Q), seed=(521,))
    d = S.conv_desc(N, C, H, W, K, R, S_, 1, pd, "fp32")
    df, db = S.sysml_conv2d_bwd_filter(m, dev(dy), d)
    dfr, dbr = oracle.conv2d_bwd_filter(x.astype(np.float64), dy, N, C, H, W, K, R, S_, (1, 1), (pd, pd))
    assert_close(host(df), dfr, 1e-4, "csr bwd_filter")
    assert_close(host(db), dbr, 1e-4, "csr db")
    df2, db2 = S.sysml_conv2d_bwd_filter(m, dev(dy), d)
    assert np.array_equal(host(df), host(df2)) and np.array_equal(host(db), host(db2))  # deterministic


def test_csr_dyadic_fused_bit_exact(S):
    N = 9
    x = synth.mnist_like_dyadic(N, seed=(510,))
    m, (rp, ci, v) = _csr_dev(S, x)
    f = synth.dyadic((32, 25), -3, 3, 16, seed=(511,))
    b = synth.dyadic((32,), -3, 3, 16, seed=(512,))
    d = S.conv_desc(N, 1, 28, 28, 32, 5, 5, 1, 2, "tf32")
    pd = S.pool_desc(N, 32, 28, 28, 2, 2, 2, 0, True)
    out, arg = S.sysml_conv2d_bias_relu_maxpool(m, dev(f), dev(b), d, pd)
    z = oracle.conv2d_fwd(x, f, N, 1, 28, 28, 32, 5, 5, (1, 1), (2, 2), bias=b)
    oref, aref = oracle.relu_maxpool(z, N, 32, 28, 28, 2, 2, (2, 2), (0, 0))
    assert np.array_equal(host(arg), aref) and np.array_equal(host(out).astype(np.float64), oref)


def test_csr_check_flags_violations(S):
    rp = np.array([0, 2, 3], np.int32)
    ci = np.array([3, 1, 0], np.int32)   # row 0 unsorted
    v = np.array([1.0, 2.0, 0.0], np.float32)  # row 1 explicit zero
    m = S.CSR(dev(rp, torch.int32), dev(ci, torch.int32), dev(v), 2, 4)
    assert S.sysml_csr_check(m) == 2


# ---------------------------------------------------------------------------- errors

def test_shape_errors_name_shapes(S):
    d = S.conv_desc(2, 1, 3, 3, 1, 5, 5, 1, 0, "fp32")
    with pytest.raises(S.SysmlError) as e:
        S.sysml_conv2d(torch.zeros(2, 9, device="cuda"), torch.zeros(1, 25, device="cuda"), d,
                       out=torch.zeros(2, 1, device="cuda"))
    assert e.value.status == 2 and "3x3" in str(e.value)
    pd = S.pool_desc(1, 1, 4, 4, 2, 2, 2, (2, 0))
    with pytest.raises(S.SysmlError) as e:
        S.sysml_relu_maxpool(torch.zeros(1, 16, device="cuda"), pd, out=torch.zeros(1, 16, device="cuda"))
    assert e.value.status == 2


# ---------------------------------------------------------------------------- LeNet step

def _lenet_case(n, dyadic=False, seed=600):
    if dyadic:
        x = synth.mnist_like_dyadic(n, seed=(seed,))
        prm = synth.lenet_params(seed=(seed + 1,), dyadic_grid=True)
    else:
        x = synth.mnist_like(n, seed=(seed,))
        prm = synth.lenet_params(seed=(seed + 1,)) + synth.normal((83466,), 0.01, seed=(seed + 2,))
    y = synth.labels(n, seed=(seed + 3,))
    return x, y, prm.astype(np.float32)


@pytest.mark.parametrize("csr", [False, True])
@pytest.mark.parametrize("math,dyadic", [("fp32", False), ("tf32", True), ("fp32", True)])
def test_lenet_fwd_bwd_parity(S, math, dyadic, csr):
    n = 10
    x, y, prm = _lenet_case(n, dyadic)
    g_ref, loss_ref = oracle.lenet_fwd_bwd(x, y, prm, n_global=32)
    net = S.LeNet(16, math=math, csr=csr, max_nnz=n * 784)
    xin = _csr_dev(S, x)[0] if csr else dev(x)
    grads = torch.empty(83466, device="cuda")
    loss = torch.empty(1, device="cuda")
    net.fwd_bwd(dev(prm), xin, dev(y, torch.int32), 32, grads, loss)
    g = host(grads)
    offs = np.cumsum([0] + [int(np.prod(s)) for _, s in synth.LENET_PARAM_SHAPES])
    for i, (name, _) in enumerate(synth.LENET_PARAM_SHAPES):
        assert_close(g[offs[i]:offs[i + 1]], g_ref[offs[i]:offs[i + 1]], TOL[math], name)
    assert abs(host(loss)[0] - loss_ref) <= 1e-5 * abs(loss_ref)


def test_lenet_step_sgd_and_determinism(S):
    n = 8
    x, y, prm = _lenet_case(n, seed=700)
    net = S.LeNet(n, math="tf32")
    results = []
    for _ in range(2):
        p = dev(prm)
        g = torch.empty(83466, device="cuda")
        net.step(p, g, dev(x), dev(y, torch.int32), n, lr=0.01)
        results.append((host(p).tobytes(), host(g)))
    assert results[0][0] == results[1][0]
    p_ref = oracle.sgd_update(prm, results[0][1], 0.01)
    assert_close(np.frombuffer(results[0][0], np.float32), p_ref, 1e-7, "sgd")
    # host-input end-to-end entry point gives the same parameters
    p = dev(prm)
    g = torch.empty(83466, device="cuda")
    loss = net.step_host(p, g, torch.from_numpy(x).pin_memory(), torch.from_numpy(y).pin_memory(), n)
    assert host(p).tobytes() == results[0][0]
    assert np.isfinite(loss)


def test_stream_k_opt_in_parity():
    """The opt-in stream-K schedule of the tcgen05 conv kernel (SYSML_TC_SK=1, read once per
    process): the conv and LeNet parity tests above, re-run in a child process with it on."""
    import os
    import subprocess
    import sys
    env = dict(os.environ, SYSML_TC_SK="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "gpu", "-p", "no:cacheprovider",
                        os.path.abspath(__file__), "-k",
                        "(test_conv_fwd_bwd_parity and tf32) or test_lenet_fwd_bwd_parity or determinism"],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


def test_phase_unfused_parity():
    """Strided R, S > 1 convs with the phase tensors materialised (SYSML_PHASE_FUSED=0: the
    X' / dX' gather kernels instead of the in-kernel gather / scatter), with the phase path
    off (SYSML_NO_PHASE=1: the FP32-SIMT kernels under TF32), with the C < 8 im2col bwd_filter
    split into 1 MB chunks (summed in chunk order) and with it off, re-run in child processes."""
    import os
    import subprocess
    import sys
    for var, val in (("SYSML_PHASE_FUSED", "0"), ("SYSML_NO_PHASE", "1"), ("SYSML_IM2COL_WS_MB", "1"),
                     ("SYSML_NO_IM2COL", "1")):
        env = dict(os.environ, **{var: val})
        r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "gpu", "-p", "no:cacheprovider",
                            os.path.abspath(__file__), "-k",
                            "(test_conv_fwd_bwd_parity and tf32) or resnet50 or (random and tf32)"],
                           env=env, capture_output=True, text=True, timeout=900)
        assert r.returncode == 0, var + ": " + r.stdout[-3000:] + r.stderr[-2000:]


def test_lenet_step_nccl_bucketed_allreduce(S):
    """sysml_lenet_step with a communicator: the bucketed allreduce overlapped on the handle's
    side stream ({F2,b2,W3,b3} after conv2 bwd_filter, {F1,b1} at the end) gives bitwise the
    same parameters as the single end-of-step allreduce and as no communicator (one rank: the
    sum is the identity), eagerly and replayed from a captured CUDA graph."""
    import os
    import socket
    import torch.distributed as dist
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        t = torch.ones(1, device="cuda")
        dist.all_reduce(t)
        comm = S.nccl_comm_ptr(allow_single=True)
        assert comm
        n = 24
        x, y, prm = _lenet_case(n, seed=910)
        net = S.LeNet(n, math="tf32")
        out = {}
        for mode in ("none", "single", "overlap"):
            os.environ["SYSML_AR_OVERLAP"] = "0" if mode == "single" else "1"
            p, g = dev(prm), torch.empty(83466, device="cuda")
            for _ in range(2):
                net.step(p, g, dev(x), dev(y, torch.int32), 64, lr=0.01,
                         nccl_comm=None if mode == "none" else comm)
            torch.cuda.synchronize()
            out[mode] = host(p).tobytes()
        assert out["overlap"] == out["single"] == out["none"]
        # captured graph (side-stream fork / join inside the capture)
        os.environ["SYSML_AR_OVERLAP"] = "1"
        p, g = dev(prm), torch.empty(83466, device="cuda")
        xd, yd = dev(x), dev(y, torch.int32)
        net.step(p, g, xd, yd, 64, lr=0.01, nccl_comm=comm)  # warm-up (plans, attributes)
        p.copy_(dev(prm))
        cs = torch.cuda.Stream()
        cs.wait_stream(torch.cuda.current_stream())
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=cs):
            net.step(p, g, xd, yd, 64, lr=0.01, nccl_comm=comm)
        torch.cuda.current_stream().wait_stream(cs)
        p.copy_(dev(prm))
        torch.cuda.synchronize()
        for _ in range(2):
            gr.replay()
        torch.cuda.synchronize()
        assert host(p).tobytes() == out["overlap"]
    finally:
        os.environ.pop("SYSML_AR_OVERLAP", None)
        dist.destroy_process_group()


OPT_KINDS = ["sgd", "momentum", "nesterov", "adagrad", "rmsprop", "adam"]


@pytest.mark.parametrize("kind", OPT_KINDS)
def test_optimizer_update_vs_oracle(S, kind):
    """sysml_optimizer_update (fp32) against oracle_optimizer_update (fp64), three steps from a
    non-zero state, n ragged (not a multiple of the block), hyper-parameters off their defaults."""
    rng = np.random.default_rng(20 + OPT_KINDS.index(kind))
    n = 1000003
    hp = dict(lr=0.013, mu=0.85, rho=0.95, eps=1e-6, beta1=0.8, beta2=0.99)
    p = rng.normal(size=n)
    nst = oracle.OPT_STATE[kind]
    st = np.abs(rng.normal(size=nst * n)) if nst else np.zeros(0)
    desc = S.optimizer_desc(kind, **hp)
    assert S.lib().sysml_optimizer_state_floats(desc.kind) == nst
    pd = dev(p)
    sd = dev(st) if nst else None
    p_ref, st_ref = p.astype(np.float32).astype(np.float64), st.astype(np.float32).astype(np.float64)
    for t in range(1, 4):
        g = rng.normal(size=n).astype(np.float32)
        S.sysml_optimizer_update(desc, pd, dev(g), sd, t=t)
        p_ref, st_ref = oracle.optimizer_update(kind, p_ref, g, st_ref if nst else np.zeros(0), t=t, **hp)
    assert_close(host(pd), p_ref, 1e-5, f"{kind} params")
    if nst:
        assert_close(host(sd), st_ref, 1e-5, f"{kind} state")


@pytest.mark.parametrize("kind", ["momentum", "adam"])
def test_lenet_step_opt_vs_oracle_update(S, kind):
    """sysml_lenet_step_opt = fwd_bwd + optimizer update: the parameters after the step equal
    the oracle optimizer applied to the gradients of the same GPU fwd_bwd."""
    n = 16
    x, y, prm = _lenet_case(n, seed=930)
    net = S.LeNet(n, math="tf32")
    desc = S.optimizer_desc(kind, lr=0.02)
    nst = oracle.OPT_STATE[kind]
    g = torch.empty(83466, device="cuda")
    net.fwd_bwd(dev(prm), dev(x), dev(y, torch.int32), 64, g)
    g_h = host(g)
    p = dev(prm)
    st = torch.zeros(nst * 83466, device="cuda")
    net.step_opt(p, torch.empty(83466, device="cuda"), st, desc, 1, dev(x), dev(y, torch.int32), 64)
    p_ref, st_ref = oracle.optimizer_update(kind, prm.astype(np.float64), g_h, np.zeros(nst * 83466), t=1,
                                            lr=0.02)
    assert_close(host(p), p_ref, 1e-5, f"{kind} step params")
    assert_close(host(st), st_ref, 1e-5, f"{kind} step state")


def test_lenet_full_batch_bench_config(S):
    """BJ configs[4] at full size, in the launch configuration bench.py times (local batch 8192,
    TF32): the 8192 images are 8 distinct images repeated 1024 times, so the oracle needs only
    the 8 -- grads = 1024 x the 8-image oracle gradient sum, both scaled by 1/8192."""
    k, rep = 8, 1024
    x8, y8, prm = _lenet_case(k, dyadic=True, seed=960)  # TF32-exact: no argmax near-tie flips
    g8, loss8 = oracle.lenet_fwd_bwd(x8, y8, prm, n_global=k * rep)
    x = np.tile(x8, (rep, 1))
    y = np.tile(y8, rep)
    net = S.LeNet(k * rep, math="tf32")
    grads = torch.empty(83466, device="cuda")
    loss = torch.zeros(1, device="cuda")
    net.fwd_bwd(dev(prm), dev(x), dev(y, torch.int32), k * rep, grads, loss)
    g = host(grads)
    offs = np.cumsum([0] + [int(np.prod(s)) for _, s in synth.LENET_PARAM_SHAPES])
    for i, (name, _) in enumerate(synth.LENET_PARAM_SHAPES):
        assert_close(g[offs[i]:offs[i + 1]], rep * g8[offs[i]:offs[i + 1]], TOL["tf32"], name + " @8192")
    assert abs(host(loss)[0] - rep * loss8) <= 1e-4 * abs(rep * loss8)


@pytest.mark.parametrize("layer", [(128, 256, 14, 14, 256, 3, 1), (128, 1024, 14, 14, 256, 1, 0)])
def test_resnet_layer_full_size_sampled(S, layer):
    """BJ configs[3] ResNet-style layers at full N = 128 (TF32): fwd and bwd_data checked on two
    sampled images (the oracle per image), bwd_filter on 96 sampled (k, c, r, s) entries, each
    the exact fp64 sum over all 128 images and P*Q positions."""
    N, C, H, W, K, R, pd = layer
    P = Q = H + 2 * pd - R + 1
    x, f, b, dy = synth.conv_problem_U(N, C, H, W, K, R, R, P, Q, seed=(970,))
    d = S.conv_desc(N, C, H, W, K, R, R, 1, pd, "tf32")
    y = host(S.sysml_conv2d(dev(x), dev(f), d, bias=dev(b))).reshape(N, -1)
    dx = host(S.sysml_conv2d_bwd_data(dev(f), dev(dy), d)).reshape(N, -1)
    df, db = S.sysml_conv2d_bwd_filter(dev(x), dev(dy), d)
    df, db = host(df).reshape(K, C, R, R), host(db)
    for n in (0, N - 1):
        yr = oracle.conv2d_fwd(x[n:n + 1], f, 1, C, H, W, K, R, R, (1, 1), (pd, pd), bias=b)
        assert_close(y[n:n + 1], yr, TOL["tf32"], f"fwd image {n}")
        dxr = oracle.conv2d_bwd_data(f, dy[n:n + 1], 1, C, H, W, K, R, R, (1, 1), (pd, pd))
        assert_close(dx[n:n + 1], dxr, TOL["tf32"], f"bwd_data image {n}")
    rng = np.random.default_rng(971)
    X = np.pad(x.astype(np.float64).reshape(N, C, H, W), ((0, 0), (0, 0), (pd, pd), (pd, pd)))
    DY = dy.astype(np.float64).reshape(N, K, P, Q)
    idx = [(rng.integers(K), rng.integers(C), rng.integers(R), rng.integers(R)) for _ in range(96)]
    ref = np.array([np.sum(DY[:, k] * X[:, c, r:r + P, s:s + Q]) for k, c, r, s in idx])
    got = np.array([df[k, c, r, s] for k, c, r, s in idx])
    assert_close(got, ref, TOL["tf32"], "bwd_filter sampled")
    assert_close(db, DY.sum(axis=(0, 2, 3)), 1e-4, "db")


@pytest.mark.parametrize("layer", [(32, 3, 224, 224, 64, 7, 2, 3),    # ResNet-50 stem
                                   (32, 128, 56, 56, 128, 3, 2, 1),   # conv3_1 3x3/2 (v1.5)
                                   (32, 512, 14, 14, 512, 3, 2, 1)])  # conv5_1 3x3/2
def test_resnet50_strided_full_size_sampled(S, layer):
    """NEXT-2: the ResNet-50 strided convs at ImageNet size, N = 32 (TF32, phase path).  fwd and
    bwd_data on two sampled images against the per-image oracle; bwd_filter on 64 sampled
    entries, each the exact fp64 sum over all images and output positions."""
    N, C, H, W, K, R, st, pd = layer
    P = Q = (H + 2 * pd - R) // st + 1
    x, f, b, dy = synth.conv_problem_U(N, C, H, W, K, R, R, P, Q, seed=(975,))
    d = S.conv_desc(N, C, H, W, K, R, R, st, pd, "tf32")
    y = host(S.sysml_conv2d(dev(x), dev(f), d, bias=dev(b))).reshape(N, -1)
    dx = host(S.sysml_conv2d_bwd_data(dev(f), dev(dy), d)).reshape(N, -1)
    df, db = S.sysml_conv2d_bwd_filter(dev(x), dev(dy), d)
    df, db = host(df).reshape(K, C, R, R), host(db)
    for n in (0, N - 1):
        yr = oracle.conv2d_fwd(x[n:n + 1], f, 1, C, H, W, K, R, R, (st, st), (pd, pd), bias=b)
        assert_close(y[n:n + 1], yr, TOL["tf32"], f"fwd image {n}")
        dxr = oracle.conv2d_bwd_data(f, dy[n:n + 1], 1, C, H, W, K, R, R, (st, st), (pd, pd))
        assert_close(dx[n:n + 1], dxr, TOL["tf32"], f"bwd_data image {n}")
    rng = np.random.default_rng(976)
    X = np.pad(x.astype(np.float64).reshape(N, C, H, W), ((0, 0), (0, 0), (pd, pd), (pd, pd)))
    DY = dy.astype(np.float64).reshape(N, K, P, Q)
    idx = [(rng.integers(K), rng.integers(C), rng.integers(R), rng.integers(R)) for _ in range(64)]
    e = (P - 1) * st + 1
    ref = np.array([np.sum(DY[:, k] * X[:, c, r:r + e:st, s:s + e:st]) for k, c, r, s in idx])
    got = np.array([df[k, c, r, s] for k, c, r, s in idx])
    assert_close(got, ref, TOL["tf32"], "bwd_filter sampled")
    assert_close(db, DY.sum(axis=(0, 2, 3)), 1e-4, "db")


def _resnet50_shapes():
    import importlib.util, os
    spec = importlib.util.spec_from_file_location(
        "resnet50_sweep", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools", "resnet50_sweep.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m.RESNET50


@pytest.mark.parametrize("name", list(_resnet50_shapes()))
def test_resnet50_every_layer_shape(S, name):
    """NEXT-2 sweep: every distinct ResNet-50 conv shape (stem, 1x1 / 3x3, stride-2 3x3 and
    1x1 downsamples, 56/28/14/7 planes) at N = 2, TF32, all three operators vs the oracle."""
    C, H, K, R, st, pd = _resnet50_shapes()[name]
    N = 2
    P = (H + 2 * pd - R) // st + 1
    x, f, b, dy = synth.conv_problem_U(N, C, H, H, K, R, R, P, P, seed=(980,))
    d = S.conv_desc(N, C, H, H, K, R, R, st, pd, "tf32")
    y = S.sysml_conv2d(dev(x), dev(f), d, bias=dev(b))
    assert_close(host(y), oracle.conv2d_fwd(x, f, N, C, H, H, K, R, R, (st, st), (pd, pd), bias=b), TOL["tf32"], "fwd")
    df, db = S.sysml_conv2d_bwd_filter(dev(x), dev(dy), d)
    dfr, dbr = oracle.conv2d_bwd_filter(x, dy, N, C, H, H, K, R, R, (st, st), (pd, pd))
    assert_close(host(df), dfr, TOL["tf32"], "bwd_filter")
    assert_close(host(db), dbr, 1e-4, "db")
    dx = S.sysml_conv2d_bwd_data(dev(f), dev(dy), d)
    assert_close(host(dx), oracle.conv2d_bwd_data(f, dy, N, C, H, H, K, R, R, (st, st), (pd, pd)), TOL["tf32"], "bwd_data")


@pytest.mark.parametrize("math", ["fp32", "tf32"])
def test_csr_all_empty_matrix(S, math):
    """Degenerate CSR input: nnz = 0 (every image empty) -> conv = bias, fused conv+pool =
    relu(bias) with the first window position as argmax, bwd_filter = 0 (db still = sum dY)."""
    N = 6
    x = np.zeros((N, 784), np.float32)
    m, _ = _csr_dev(S, x)
    assert m.nnz == 0
    f = synth.normal((32, 25), 0.2, seed=(980,))
    b = synth.normal((32,), 0.1, seed=(981,))
    d = S.conv_desc(N, 1, 28, 28, 32, 5, 5, 1, 2, math)
    y = host(S.sysml_conv2d(m, dev(f), d, bias=dev(b)))
    assert_close(y, np.repeat(b.astype(np.float64), 784)[None, :].repeat(N, 0), TOL[math], "empty csr fwd")
    dy = synth.normal((N, 32 * 784), seed=(982,))
    df, db = S.sysml_conv2d_bwd_filter(m, dev(dy), d)
    assert not np.any(host(df))
    assert_close(host(db), dy.astype(np.float64).reshape(N, 32, 784).sum(axis=(0, 2)), 1e-4, "empty csr db")
    pd = S.pool_desc(N, 32, 28, 28, 2, 2, 2, 0, True)
    out, arg = S.sysml_conv2d_bias_relu_maxpool(m, dev(f), dev(b), d, pd)
    z = np.repeat(b.astype(np.float64), 784)[None, :].repeat(N, 0)
    oref, aref = oracle.relu_maxpool(z, N, 32, 28, 28, 2, 2, (2, 2), (0, 0))
    assert_close(host(out), oref, TOL[math], "empty csr fused")
    assert np.array_equal(host(arg), aref)


def test_lenet_step_host_pipelined_matches_step_host(S):
    """The pipelined host-input step (next batch copied while this step computes) gives bitwise
    the same parameters and losses as the plain host step, over rotating batches and with a
    prefetch miss (a batch other than the one prefetched)."""
    n = 32
    batches = []
    for k in range(3):
        x, y, prm = _lenet_case(n, seed=990 + 10 * k)
        batches.append((torch.from_numpy(x).pin_memory(), torch.from_numpy(y).pin_memory()))
    prm = _lenet_case(n, seed=990)[2]
    order = [0, 1, 2, 0]  # step 3 runs batch 0 while batch 2 was... prefetched as the next of step 2
    net = S.LeNet(n, math="tf32")
    p1, g1 = dev(prm), torch.empty(83466, device="cuda")
    l1 = [net.step_host(p1, g1, batches[b][0], batches[b][1], n) for b in order]
    net2 = S.LeNet(n, math="tf32")
    p2, g2 = dev(prm), torch.empty(83466, device="cuda")
    l2 = []
    for i, b in enumerate(order):
        nb = order[i + 1] if i + 1 < len(order) else None
        if i == 2:
            nb = 1  # prefetch a batch the next call does not use -> a miss at step 3
        l2.append(net2.step_host_pipelined(p2, g2, batches[b][0], batches[b][1], n,
                                           next_x=batches[nb][0] if nb is not None else None,
                                           next_labels=batches[nb][1] if nb is not None else None))
    assert l1 == l2
    assert host(p1).tobytes() == host(p2).tobytes()


SF_SHAPES = [  # N, C, H, W, K, R, S, stride, pad, filter density
    (6, 1, 28, 28, 32, 5, 5, 1, 2, 0.3),
    (3, 4, 9, 7, 6, 3, 3, 2, 1, 0.5),
    (2, 16, 8, 8, 40, 1, 1, 1, 0, 0.2),
    (2, 2, 6, 5, 3, 4, 2, 1, (2, 0), 1.0),
    (2, 64, 14, 14, 20, 3, 3, 1, 1, 0.05),   # > SF_CHUNK-sized filter rows are not needed: 576 cols
]


@pytest.mark.parametrize("csr_input", [False, True])
@pytest.mark.parametrize("shape", SF_SHAPES)
def test_conv2d_csr_filter_vs_oracle(S, shape, csr_input):
    """Dense input / sparse filter and sparse input / sparse filter against
    oracle_conv2d_fwd_csr_filter (fp32 tolerance); includes an empty filter row."""
    N, C, H, W, K, R, S_, st, pd, dens = shape
    pd = pd if isinstance(pd, tuple) else (pd, pd)
    rng = np.random.default_rng(40 + SF_SHAPES.index(shape))
    x = synth.uniform((N, C * H * W), -1.0, 1.0, seed=(41,))
    if csr_input:
        x[rng.random(x.shape) > 0.25] = 0.0
    f = rng.normal(size=(K, C * R * S_)).astype(np.float32)
    f[rng.random(f.shape) > dens] = 0.0
    f[0] = 0.0
    b = rng.normal(size=K).astype(np.float32)
    frp, fci, fv = synth.to_csr(f)
    fc = S.CSR(dev(frp, torch.int32), dev(fci, torch.int32), dev(fv), K, C * R * S_)
    xin = _csr_dev(S, x)[0] if csr_input else dev(x)
    d = S.conv_desc(N, C, H, W, K, R, S_, st, pd, "fp32")
    y = S.sysml_conv2d_csr_filter(xin, fc, d, bias=dev(b))
    ref = oracle.conv2d_fwd_csr_filter(x.astype(np.float32).astype(np.float64), frp, fci, fv, N, C, H, W, K,
                                       R, S_, (st, st), pd, bias=b)
    assert_close(host(y), ref, 1e-4, "sparse-filter conv")
    y2 = S.sysml_conv2d_csr_filter(xin, fc, d, bias=dev(b))
    assert np.array_equal(host(y), host(y2))  # stored-order sums: deterministic


def test_decide_format_and_dense_to_csr(S):
    """GPU non-zero count and dense -> CSR: bit-exact against the
    re-encoding in synth, the 0.4 threshold, empty rows, and the densify round trip."""
    x = synth.mnist_like(37, seed=(700,))
    x[3] = 0.0
    x[5, :] = -0.0
    nnz = int(np.count_nonzero(x))
    xd = dev(x)
    assert S.sysml_count_nonzeros(xd) == nnz == oracle.decide_format(x)[1]
    m = S.dense_to_csr(xd)
    rp, ci, v = synth.to_csr(x)
    assert np.array_equal(host(m.row_ptr), rp) and np.array_equal(host(m.col_idx), ci)
    assert np.array_equal(host(m.val), v)
    assert np.array_equal(oracle.csr_densify(host(m.row_ptr), host(m.col_idx), host(m.val), 37, 784),
                          x.astype(np.float64))
    assert isinstance(S.decide_format(xd), S.CSR) and oracle.decide_format(x)[0] == "sparse"  # MNIST ~0.19
    dense = dev(synth.uniform((8, 50), 0.5, 1.0, seed=(701,)))
    assert S.decide_format(dense) is dense
    a = np.zeros((10, 10), np.float32)
    a.flat[:40] = 1.0
    assert isinstance(S.decide_format(dev(a)), S.CSR)  # nnz/size = 0.4 -> sparse
    a.flat[40] = 1.0
    assert not isinstance(S.decide_format(dev(a)), S.CSR)


@pytest.mark.parametrize("csr", [False, True])
@pytest.mark.parametrize("math", ["fp32", "tf32"])
def test_lenet_predict_vs_oracle(S, math, csr):
    """Scoring (sysml_lenet_predict) against the oracle forward's softmax / argmax: dyadic
    inputs, so TF32 logits are exact and the labels must match exactly."""
    n = 40
    x, _, prm = _lenet_case(n, dyadic=True, seed=1010)
    net = S.LeNet(64, math=math, csr=csr, max_nnz=n * 784)
    xin = _csr_dev(S, x)[0] if csr else dev(x)
    pred, probs = net.predict(dev(prm), xin, probs=True)
    pred_ref, probs_ref = oracle.lenet_predict(x, prm)
    assert np.array_equal(host(pred), pred_ref)
    assert_close(host(probs), probs_ref, TOL[math], "probs")
    assert np.array_equal(host(net.predict(dev(prm), xin)), pred_ref)


def _random_conv_shapes(count, seed):
    rng = np.random.default_rng(seed)
    shapes = []
    while len(shapes) < count:
        N = int(rng.integers(1, 5))
        C = int(rng.choice([1, 2, 3, 8, 13, 16, 24, 40, 64]))
        K = int(rng.choice([1, 5, 16, 17, 32, 48, 64, 96, 130]))
        R = int(rng.choice([1, 2, 3, 5]))
        S_ = int(rng.choice([1, 3, 5])) if rng.random() < 0.7 else R
        st = int(rng.choice([1, 1, 1, 2]))
        ph, pw = int(rng.integers(0, R)), int(rng.integers(0, S_))
        H, W = int(rng.integers(R, 19)), int(rng.integers(S_, 19))
        if (H + 2 * ph - R) // st + 1 < 1 or (W + 2 * pw - S_) // st + 1 < 1:
            continue
        shapes.append((N, C, H, W, K, R, S_, st, (ph, pw)))
    return shapes


@pytest.mark.parametrize("math", ["fp32", "tf32"])
@pytest.mark.parametrize("shape", _random_conv_shapes(24, 2026))
def test_conv_random_shape_sweep(S, shape, math):
    """Seeded random sweep over conv shapes (strides, pads, rectangular kernels, odd sizes,
    channel / filter counts around tile boundaries): fwd (+bias), bwd_filter (+db) and bwd_data
    against the oracle -- guards the plan / dispatch corners of every kernel family."""
    (N, C, H, W, K, R, S_, st, pd, P, Q), x, f, b, dy = _conv_case(shape, 77)
    d = S.conv_desc(N, C, H, W, K, R, S_, st, pd, math)
    y = S.sysml_conv2d(dev(x), dev(f), d, bias=dev(b))
    assert_close(host(y), oracle.conv2d_fwd(x, f, N, C, H, W, K, R, S_, st, pd, bias=b), TOL[math], "fwd")
    df, db = S.sysml_conv2d_bwd_filter(dev(x), dev(dy), d)
    dfr, dbr = oracle.conv2d_bwd_filter(x, dy, N, C, H, W, K, R, S_, st, pd)
    assert_close(host(df), dfr, TOL[math], "bwd_filter")
    assert_close(host(db), dbr, 1e-4, "db")
    dx = S.sysml_conv2d_bwd_data(dev(f), dev(dy), d)
    assert_close(host(dx), oracle.conv2d_bwd_data(f, dy, N, C, H, W, K, R, S_, st, pd), TOL[math], "bwd_data")


@pytest.mark.parametrize("math", ["fp32", "tf32"])
@pytest.mark.parametrize("shape", _random_conv_shapes(32, 4242))
def test_conv_random_shape_sweep_b(S, shape, math):
    """Second seed of the random conv-shape sweep."""
    test_conv_random_shape_sweep(S, shape, math)


def _random_pool_shapes(count, seed):
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < count:
        N = int(rng.integers(1, 5))
        C = int(rng.choice([1, 3, 8, 16, 32]))
        K = int(rng.choice([5, 16, 32, 48, 64]))
        R = int(rng.choice([3, 5]))
        pad = R // 2
        H, W = 2 * int(rng.integers(2, 10)), 2 * int(rng.integers(2, 10))
        out.append((N, C, H, W, K, R, pad))
    return out


@pytest.mark.parametrize("math", ["fp32", "tf32"])
@pytest.mark.parametrize("shape", _random_pool_shapes(16, 99))
def test_fused_conv_pool_random_sweep(S, shape, math):
    """Random fused conv + bias + relu + 2x2/2 max-pool shapes on dyadic inputs (exact in TF32):
    pooled values and int32 argmax bit-exact against the oracle."""
    N, C, H, W, K, R, pad = shape
    x = synth.dyadic((N, C * H * W), -2, 2, 8, seed=(91,))
    f = synth.dyadic((K, C * R * R), -2, 2, 8, seed=(92,))
    b = synth.dyadic((K,), -2, 2, 8, seed=(93,))
    d = S.conv_desc(N, C, H, W, K, R, R, 1, pad, math)
    pd = S.pool_desc(N, K, H, W, 2, 2, 2, 0, True)
    out, arg = S.sysml_conv2d_bias_relu_maxpool(dev(x), dev(f), dev(b), d, pd)
    z = oracle.conv2d_fwd(x, f, N, C, H, W, K, R, R, (1, 1), (pad, pad), bias=b)
    oref, aref = oracle.relu_maxpool(z, N, K, H, W, 2, 2, (2, 2), (0, 0))
    assert np.array_equal(host(out).astype(np.float64), oref)
    assert np.array_equal(host(arg), aref)


@pytest.mark.parametrize("math", ["fp32", "tf32"])
@pytest.mark.parametrize("N,K,R", [(1, 5, 3), (7, 16, 5), (33, 32, 5), (5, 32, 3), (130, 32, 5)])
def test_csr_conv1_random_sweep(S, N, K, R, math):
    """CSR conv1-style inputs (C = 1, 28x28, ~19% dense) over batch sizes and filter counts:
    fwd, bwd_filter and the fused conv+pool against the oracle."""
    x = synth.mnist_like(N, seed=(95, N))
    m, (rp, ci, v) = _csr_dev(S, x)
    xd = oracle.csr_densify(rp, ci, v, N, 784)
    pad = R // 2
    f = synth.normal((K, R * R), 0.3, seed=(96,))
    b = synth.normal((K,), 0.1, seed=(97,))
    d = S.conv_desc(N, 1, 28, 28, K, R, R, 1, pad, math)
    y = S.sysml_conv2d(m, dev(f), d, bias=dev(b))
    assert_close(host(y), oracle.conv2d_fwd(xd, f, N, 1, 28, 28, K, R, R, (1, 1), (pad, pad), bias=b), TOL[math], "fwd")
    dy = synth.normal((N, K * 784), seed=(98,))
    df, db = S.sysml_conv2d_bwd_filter(m, dev(dy), d)
    dfr, dbr = oracle.conv2d_bwd_filter(xd, dy, N, 1, 28, 28, K, R, R, (1, 1), (pad, pad))
    assert_close(host(df), dfr, 1e-4, "bwd_filter")
    assert_close(host(db), dbr, 1e-4, "db")
    pd = S.pool_desc(N, K, 28, 28, 2, 2, 2, 0, True)
    out, arg = S.sysml_conv2d_bias_relu_maxpool(m, dev(f), dev(b), d, pd)
    z = oracle.conv2d_fwd(xd, f, N, 1, 28, 28, K, R, R, (1, 1), (pad, pad), bias=b)
    oref, aref = oracle.relu_maxpool(z, N, K, 28, 28, 2, 2, (2, 2), (0, 0))
    assert_close(host(out), oref, TOL[math], "fused")
    a = host(arg)
    assert_argmax_in_window(a, K, 28, 28, 14, 14, 2, 2, (2, 2))
    flips = assert_valid_argmax(a, z, oref, TOL[math], "fused", exact_ref=aref)
    print(f"csr sweep {math} N={N} K={K} R={R}: {flips} argmax flips of {a.size} windows")


@pytest.mark.parametrize("n", [1, 3, 31, 33, 65, 130])
def test_lenet_fwd_bwd_batch_sweep(S, n):
    """LeNet fwd_bwd (TF32, dyadic) over ragged local batch sizes: odd counts (F3 sample pairs),
    non-multiples of 32 (B2p chunks, B1 CTAs, dW3 chunks) and a handle larger than the batch."""
    x, y, prm = _lenet_case(n, dyadic=True, seed=1100 + n)
    g_ref, loss_ref = oracle.lenet_fwd_bwd(x, y, prm, n_global=2 * n)
    net = S.LeNet(n + 7, math="tf32")
    grads = torch.empty(83466, device="cuda")
    loss = torch.empty(1, device="cuda")
    net.fwd_bwd(dev(prm), dev(x), dev(y, torch.int32), 2 * n, grads, loss)
    g = host(grads)
    offs = np.cumsum([0] + [int(np.prod(s)) for _, s in synth.LENET_PARAM_SHAPES])
    for i, (name, _) in enumerate(synth.LENET_PARAM_SHAPES):
        assert_close(g[offs[i]:offs[i + 1]], g_ref[offs[i]:offs[i + 1]], TOL["tf32"], f"{name} n={n}")
    assert abs(host(loss)[0] - loss_ref) <= 1e-5 * abs(loss_ref)
