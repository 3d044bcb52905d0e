"""GPU parity of the LeNet-512 step (NEXT-4: affine 3136->512 + relu + inverted dropout +
affine 512->10; R22-R24) against the fp64 oracle, through the C ABI.

Protocol (extended to the hidden layer):
  * FP32 mode on continuous MNIST-shaped data at 1e-4 (every parameter block);
  * TF32 mode on dyadic-grid conv inputs/parameters (the fused pool argmax is exact) with the
    hidden bias offset so that no hidden unit sits within TF32 rounding of the relu kink
    (asserted on the oracle's z3): a kink flip is a legitimate TF32 outcome that would move a
    whole sample's contribution, exactly as an argmax flip does in the pools;
  * the dropout mask is the oracle's (Philox4x64-10, R23) bit for bit: any flipped unit moves
    dW4 / db3 far outside tolerance, and keep_p = 1 must equal the no-dropout network;
  * the device step counter advances once per step (graph replays included) and the mask
    follows the global row (two shards with row0 offsets sum to the full batch).
"""
import numpy as np
import pytest
import torch

import oracle
import synth

from tests.test_gpu_parity import TOL, S, assert_close, dev, host  # noqa: F401

pytestmark = pytest.mark.gpu

H = synth.LENET512_HIDDEN
NP = synth.LENET512_NUM_PARAMS
OFFS = np.cumsum([0] + [int(np.prod(s)) for _, s in synth.LENET512_PARAM_SHAPES])
NAMES = [nm for nm, _ in synth.LENET512_PARAM_SHAPES]


def _case(n, math, seed=700):
    if math == "tf32":
        x = synth.mnist_like_dyadic(n, seed=(seed,))
        prm = synth.lenet512_params(seed=(seed + 1,), dyadic_grid=True)
        # continuous hidden / output weights (the GEMMs round them to TF32 anyway)
        cont = synth.lenet512_params(seed=(seed + 2,))
        prm[OFFS[4]:OFFS[5]] = cont[OFFS[4]:OFFS[5]]
        prm[OFFS[6]:OFFS[7]] = cont[OFFS[6]:OFFS[7]]
        # hidden bias: unit u is active for every sample (s_u = +1) or dead for every sample
        # (s_u = -1), 5% of the largest |a2 W3^T| away from the kink; built from the ORACLE's
        # forward of these inputs (test-input construction, no GPU value involved)
        prm[OFFS[5]:OFFS[6]] = 0.0
        raw = oracle.lenet512_forward(x, prm)["z3"]
        big = np.abs(raw).max()
        sgn = np.where(synth.rng(seed + 4).random(H) < 0.7, 1.0, -1.0)
        prm[OFFS[5]:OFFS[6]] = sgn * (np.abs(raw).max(axis=0) + 0.05 * big)
    else:
        x = synth.mnist_like(n, seed=(seed,))
        prm = synth.lenet512_params(seed=(seed + 1,)) + synth.normal((NP,), 0.01, seed=(seed + 2,))
    y = synth.labels(n, seed=(seed + 3,))
    return x, y, prm.astype(np.float32)


def _z3_margin(x, prm):
    fw = oracle.lenet512_forward(x, prm)
    z = fw["z3"]
    return np.abs(z).min() / np.abs(z).max()


def _run_fwd_bwd(S, x, y, prm, math, n_global, keep, seed, step, row0=0, csr=False, net=None):
    n = x.shape[0]
    if net is None:
        net = S.LeNet(max(n, 8), math=math, csr=csr, max_nnz=n * 784, model="lenet512", keep_p=keep, seed=seed)
    net.set_dropout(row0=row0, step=step)
    if csr:
        rp, ci, v = synth.to_csr(x)
        xin = S.CSR(dev(rp, torch.int32), dev(ci, torch.int32), dev(v), n, 784)
    else:
        xin = dev(x)
    grads = torch.empty(NP, device="cuda")
    loss = torch.empty(1, device="cuda")
    net.fwd_bwd(dev(prm), xin, dev(y, torch.int32), n_global, grads, loss)
    torch.cuda.synchronize()
    return host(grads).astype(np.float64), float(host(loss)[0]), net


def _check_blocks(g, g_ref, tol, what):
    for i, name in enumerate(NAMES):
        assert_close(g[OFFS[i]:OFFS[i + 1]], g_ref[OFFS[i]:OFFS[i + 1]], tol, f"{what} {name}")


def test_handle_num_params(S):
    net = S.LeNet(8, model="lenet512")
    assert net.num_params == NP == S.lib().sysml_lenet512_num_params()
    assert S.LeNet(8).num_params == 83466


@pytest.mark.parametrize("csr", [False, True])
@pytest.mark.parametrize("math", ["fp32", "tf32"])
def test_lenet512_fwd_bwd_parity(S, math, csr):
    n, keep, seed, step, row0 = 37, 0.5, 11, 3, 5   # ragged: 37 rows, 2 route chunks, ldt 40
    x, y, prm = _case(n, math)
    if math == "tf32":
        assert _z3_margin(x, prm) > 0.02   # no hidden unit within TF32 reach of the relu kink
    g_ref, loss_ref = oracle.lenet512_fwd_bwd(x, y, prm, seed, step, keep, n_global=64, row0=row0)
    g, loss, _ = _run_fwd_bwd(S, x, y, prm, math, 64, keep, seed, step, row0=row0, csr=csr)
    _check_blocks(g, g_ref, TOL[math], f"{math} csr={csr}")
    assert abs(loss - loss_ref) <= (1e-5 if math == "fp32" else TOL[math]) * abs(loss_ref)


def test_lenet512_keep_one_is_the_network_without_dropout(S):
    # keep_p = 1: every unit kept, scale 1 -> the gradient of the plain relu network
    n = 20
    x, y, prm = _case(n, "fp32", seed=710)
    g_ref, _ = oracle.lenet512_fwd_bwd(x, y, prm, 0, 0, 1.0)
    g, _, _ = _run_fwd_bwd(S, x, y, prm, "fp32", n, 1.0, 123, 9)
    _check_blocks(g, g_ref, TOL["fp32"], "keep_p=1")


def test_lenet512_mask_bits_match_oracle_keep_075(S):
    # a single flipped mask bit moves one sample's contribution to a db3 entry by a whole
    # term; at n = 4 that is far above the 1e-4 tolerance (checked on the oracle itself)
    n, keep, seed, step = 4, 0.75, 2024, 17
    x, y, prm = _case(n, "fp32", seed=720)
    g_ref, _ = oracle.lenet512_fwd_bwd(x, y, prm, seed, step, keep)
    g_other, _ = oracle.lenet512_fwd_bwd(x, y, prm, seed, step + 1, keep)
    scale = np.abs(g_ref[OFFS[5]:OFFS[6]]).max()
    assert np.abs(g_other[OFFS[5]:OFFS[6]] - g_ref[OFFS[5]:OFFS[6]]).max() > 1e-2 * scale
    g, _, _ = _run_fwd_bwd(S, x, y, prm, "fp32", n, keep, seed, step)
    _check_blocks(g, g_ref, TOL["fp32"], "keep 0.75")


def test_lenet512_shards_with_row_offsets_sum_to_full_batch(S):
    # S:499 with the mask following the global row: rank 0 rows [0, 16), rank 1 rows [16, 40)
    n, keep, seed, step = 40, 0.5, 5, 2
    x, y, prm = _case(n, "fp32", seed=730)
    g_ref, _ = oracle.lenet512_fwd_bwd(x, y, prm, seed, step, keep, n_global=n)
    ga, _, _ = _run_fwd_bwd(S, x[:16], y[:16], prm, "fp32", n, keep, seed, step, row0=0)
    gb, _, _ = _run_fwd_bwd(S, x[16:], y[16:], prm, "fp32", n, keep, seed, step, row0=16)
    _check_blocks(ga + gb, g_ref, TOL["fp32"], "shard sum")


@pytest.mark.parametrize("math", ["fp32", "tf32"])
def test_lenet512_step_counter_sgd_and_graph_replay(S, math):
    n, keep, seed = 24, 0.5, 77
    x, y, prm = _case(n, math, seed=740)
    net = S.LeNet(n, math=math, model="lenet512", keep_p=keep, seed=seed)
    net.set_dropout(row0=0, step=10)
    assert net.dropout_step() == 10
    p = dev(prm)
    grads = torch.empty(NP, device="cuda")
    xd, yd = dev(x), dev(y, torch.int32)
    # TF32 parity is gated on dyadic conv parameters only (SURVEY §8(c) protocol 3), so the
    # TF32 variant keeps them with lr = 0; the FP32 variant checks the SGD update itself
    lr = 0.01 if math == "fp32" else 0.0
    net.step(p, grads, xd, yd, n, lr=lr)
    torch.cuda.synchronize()
    assert net.dropout_step() == 11
    g_ref, _ = oracle.lenet512_fwd_bwd(x, y, prm, seed, 10, keep)
    _check_blocks(host(grads).astype(np.float64), g_ref, TOL[math], "step 10")
    p_ref = oracle.sgd_update(prm, host(grads), lr)
    assert np.abs(host(p) - p_ref).max() <= 1e-6
    # CUDA-graph capture of the whole step; each replay draws the next step's mask
    s = torch.cuda.Stream()
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        net.step(p, grads, xd, yd, n, lr=0.0, stream=s)  # warm-up (step 11, lr 0: p unchanged)
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            net.step(p, grads, xd, yd, n, lr=0.0, stream=s)
    torch.cuda.synchronize()
    assert net.dropout_step() == 12   # capture launches nothing
    for t in (12, 13):
        g.replay()
        torch.cuda.synchronize()
        g_ref, _ = oracle.lenet512_fwd_bwd(x, y, host(p), seed, t, keep)  # lr 0: params fixed
        _check_blocks(host(grads).astype(np.float64), g_ref, TOL[math], f"replay step {t}")
    assert net.dropout_step() == 14


@pytest.mark.parametrize("math", ["fp32", "tf32"])
def test_lenet512_predict_vs_oracle(S, math):
    n = 50
    x, _, prm = _case(n, math, seed=750)
    pred_ref, probs_ref = oracle.lenet512_predict(x, prm)
    net = S.LeNet(64, math=math, model="lenet512", keep_p=0.5, seed=1)
    pred, probs = net.predict(dev(prm), dev(x), probs=True)
    pr = host(probs)
    assert_close(pr, probs_ref, TOL[math], "probs")
    srt = np.sort(probs_ref, axis=1)
    clear = (srt[:, -1] - srt[:, -2]) > 4 * TOL[math]   # labels exact where the oracle is decided
    np.testing.assert_array_equal(host(pred)[clear], pred_ref[clear])
    assert clear.mean() > 0.5


def test_lenet512_tf32_multi_tile_batch(S):
    # 300 rows: three 128-row M tiles of the hidden GEMM (ragged), 10 route chunks
    n, keep, seed, step = 300, 0.5, 3, 1
    x, y, prm = _case(n, "tf32", seed=760)
    assert _z3_margin(x, prm) > 0.02
    g_ref, loss_ref = oracle.lenet512_fwd_bwd(x, y, prm, seed, step, keep, n_global=512, row0=1000)
    g, loss, _ = _run_fwd_bwd(S, x, y, prm, "tf32", 512, keep, seed, step, row0=1000)
    _check_blocks(g, g_ref, TOL["tf32"], "n=300")
    assert abs(loss - loss_ref) <= TOL["tf32"] * abs(loss_ref)


@pytest.mark.parametrize("math", ["fp32", "tf32"])
@pytest.mark.parametrize("M,N,K,relu", [(37, 512, 3136, True), (300, 40, 20, False), (5, 16, 4, True),
                                        (129, 3136, 512, False)])
def test_affine_vs_oracle_definition(S, math, M, N, K, relu):
    # out = x W^T + b, relu (R7); the oracle's definition is the fp64 matmul
    x = synth.uniform((M, K), seed=(780, M)).astype(np.float32)
    W = synth.uniform((N, K), seed=(781, N)).astype(np.float32)
    b = synth.uniform((N,), seed=(782, K)).astype(np.float32)
    ref = x.astype(np.float64) @ W.astype(np.float64).T + b
    if relu:
        ref = np.maximum(ref, 0.0)
    out = S.sysml_affine(dev(x), dev(W), dev(b), relu=relu, math=math)
    assert_close(host(out), ref, TOL[math], f"affine {math} {M}x{N}x{K}")
