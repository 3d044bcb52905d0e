"""fp64 CPU oracle for the conv2d-family hot path of arXiv 1802.04647.

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference``) may import this
package.  The product library (``paper_1802_04647_b200``) never imports it and
shares no code with it.

The arithmetic lives in ``oracle/oracle.c`` (plain C, double precision, direct
nested loops, each function citing the PAPER.md / SPEC.md passage it follows).
This module is a ctypes shim: it converts inputs to float64, calls the C
function, and returns float64 numpy arrays.

Parity status per function: every function below is
pinned by tests in ``tests/test_oracle_*.py`` against worked examples, torch
fp64 library routines, adjoint identities, finite differences or brute force.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.c")


def build(force: bool = False) -> str:
    """Compile liboracle.so (gcc -O2, OpenMP, no fast-math)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-fopenmp", "-fPIC", "-shared",
               "-fno-fast-math", "-ffp-contract=off", _SRC, "-o", _SO + ".tmp", "-lm"]
        subprocess.check_call(cmd)
        os.replace(_SO + ".tmp", _SO)
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(_SO)
        i64, dp, ip = ctypes.c_int64, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int32)
        _lib.oracle_out_extent.restype = i64
        _lib.oracle_out_extent.argtypes = [i64] * 4
        _lib.oracle_conv2d_fwd.argtypes = [i64] * 11 + [dp, dp, dp, dp]
        _lib.oracle_bias_add.argtypes = [i64, i64, i64, dp, dp]
        _lib.oracle_conv2d_bwd_filter.argtypes = [i64] * 11 + [dp, dp, dp, dp]
        _lib.oracle_conv2d_bwd_data.argtypes = [i64] * 11 + [dp, dp, dp]
        _lib.oracle_relu_maxpool.argtypes = [i64] * 11 + [dp, dp, ip]
        _lib.oracle_maxpool_bwd.argtypes = [i64] * 6 + [ip, dp, dp, dp]
        _lib.oracle_csr_densify.argtypes = [i64, i64, ip, ip, dp, dp]
        _lib.oracle_lenet_num_params.restype = i64
        _lib.oracle_lenet_forward.argtypes = [i64, dp, dp, dp, ip, dp, ip, dp]
        _lib.oracle_lenet_fwd_bwd.argtypes = [i64, i64, dp, ip, dp, dp, dp]
        _lib.oracle_lenet_predict.argtypes = [i64, dp, dp, ip, dp]
        _lib.oracle_sgd_update.argtypes = [i64, dp, dp, ctypes.c_double]
        _lib.oracle_optimizer_update.argtypes = [i64, i64, dp, dp, dp] + [ctypes.c_double] * 6 + [i64]
        _lib.oracle_conv2d_fwd_csr_filter.argtypes = [i64] * 11 + [dp, ip, ip, dp, dp, dp]
        _lib.oracle_count_nonzeros.restype = i64
        _lib.oracle_count_nonzeros.argtypes = [i64, dp]
        u64, u8p = ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint8)
        _lib.oracle_philox_raw.argtypes = [u64, u64, i64, i64, ctypes.POINTER(ctypes.c_uint64)]
        _lib.oracle_dropout_mask.argtypes = [u64, u64, i64, i64, i64, ctypes.c_double, u8p]
        _lib.oracle_dropout_fwd.argtypes = [i64, dp, u8p, ctypes.c_double, dp]
        _lib.oracle_dropout_bwd.argtypes = [i64, dp, u8p, ctypes.c_double, dp]
        _lib.oracle_lenet512_num_params.restype = i64
        _lib.oracle_lenet512_forward.argtypes = [i64, i64, dp, dp, i64, u64, u64, ctypes.c_double,
                                                 dp, ip, dp, ip, dp, dp, u8p, dp]
        _lib.oracle_lenet512_fwd_bwd.argtypes = [i64, i64, i64, dp, ip, dp, u64, u64, ctypes.c_double,
                                                 dp, dp]
        _lib.oracle_lenet512_predict.argtypes = [i64, dp, dp, ip, dp]
    return _lib


def _d(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _p(a):
    if a is None:
        return None
    if a.dtype == np.int32:
        return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
    if a.dtype == np.uint8:
        return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))
    if a.dtype == np.uint64:
        return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def out_extent(n, pad, k, stride) -> int:
    return int(lib().oracle_out_extent(n, pad, k, stride))


def conv2d_fwd(x, f, N, C, H, W, K, R, S, stride=(1, 1), pad=(0, 0), bias=None):
    P, Q = out_extent(H, pad[0], R, stride[0]), out_extent(W, pad[1], S, stride[1])
    x, f = _d(x), _d(f)
    b = None if bias is None else _d(bias)
    y = np.empty((N, K * P * Q), dtype=np.float64)
    lib().oracle_conv2d_fwd(N, C, H, W, K, R, S, stride[0], stride[1], pad[0], pad[1],
                            _p(x), _p(f), _p(b), _p(y))
    return y


def bias_add(y, b, N, K, PQ):
    y = _d(y).copy()
    b = _d(b)
    lib().oracle_bias_add(N, K, PQ, _p(y), _p(b))
    return y


def conv2d_bwd_filter(x, dy, N, C, H, W, K, R, S, stride=(1, 1), pad=(0, 0)):
    x, dy = _d(x), _d(dy)
    df = np.empty((K, C * R * S), dtype=np.float64)
    db = np.empty((K,), dtype=np.float64)
    lib().oracle_conv2d_bwd_filter(N, C, H, W, K, R, S, stride[0], stride[1], pad[0], pad[1],
                                   _p(x), _p(dy), _p(df), _p(db))
    return df, db


def conv2d_bwd_data(f, dy, N, C, H, W, K, R, S, stride=(1, 1), pad=(0, 0)):
    f, dy = _d(f), _d(dy)
    dx = np.empty((N, C * H * W), dtype=np.float64)
    lib().oracle_conv2d_bwd_data(N, C, H, W, K, R, S, stride[0], stride[1], pad[0], pad[1],
                                 _p(f), _p(dy), _p(dx))
    return dx


def relu_maxpool(x, N, C, H, W, R, S, stride=(1, 1), pad=(0, 0), relu=True):
    P, Q = out_extent(H, pad[0], R, stride[0]), out_extent(W, pad[1], S, stride[1])
    x = _d(x)
    out = np.empty((N, C * P * Q), dtype=np.float64)
    arg = np.empty((N, C * P * Q), dtype=np.int32)
    lib().oracle_relu_maxpool(N, C, H, W, R, S, stride[0], stride[1], pad[0], pad[1],
                              int(bool(relu)), _p(x), _p(out), _p(arg))
    return out, arg


def maxpool_bwd(argmax, dout, N, C, H, W, P, Q, out_mask=None):
    argmax, dout = _i(argmax), _d(dout)
    m = None if out_mask is None else _d(out_mask)
    dx = np.empty((N, C * H * W), dtype=np.float64)
    lib().oracle_maxpool_bwd(N, C, H, W, P, Q, _p(argmax), _p(dout), _p(m), _p(dx))
    return dx


def csr_densify(row_ptr, col_idx, val, rows, cols):
    rp, ci, v = _i(row_ptr), _i(col_idx), _d(val)
    out = np.empty((rows, cols), dtype=np.float64)
    lib().oracle_csr_densify(rows, cols, _p(rp), _p(ci), _p(v), _p(out))
    return out


def lenet_num_params() -> int:
    return int(lib().oracle_lenet_num_params())


def lenet_forward(x, params):
    n = x.shape[0]
    x, prm = _d(x), _d(params)
    a1 = np.empty((n, 6272)); i1 = np.empty((n, 6272), dtype=np.int32)
    a2 = np.empty((n, 3136)); i2 = np.empty((n, 3136), dtype=np.int32)
    sc = np.empty((n, 10))
    lib().oracle_lenet_forward(n, _p(x), _p(prm), _p(a1), _p(i1), _p(a2), _p(i2), _p(sc))
    return dict(a1=a1, i1=i1, a2=a2, i2=i2, scores=sc)


def lenet_predict(x, params):
    """Scoring: (first maximal class, softmax probabilities) of the oracle
    forward's scores, computed in oracle.c (oracle_lenet_predict)."""
    n = x.shape[0]
    x, prm = _d(x), _d(params)
    pred = np.empty(n, dtype=np.int32)
    probs = np.empty((n, 10), dtype=np.float64)
    lib().oracle_lenet_predict(n, _p(x), _p(prm), _p(pred), _p(probs))
    return pred, probs


def lenet_fwd_bwd(x, labels, params, n_global=None):
    """Returns (grads float64[83466] pre-scaled by 1/n_global, loss_sum)."""
    n = x.shape[0]
    n_global = n if n_global is None else n_global
    x, lab, prm = _d(x), _i(labels), _d(params)
    g = np.empty(prm.size, dtype=np.float64)
    loss = ctypes.c_double(0.0)
    lib().oracle_lenet_fwd_bwd(n, n_global, _p(x), _p(lab), _p(prm), _p(g),
                               ctypes.cast(ctypes.pointer(loss), ctypes.POINTER(ctypes.c_double)))
    return g, loss.value


OPTIMIZERS = {"sgd": 0, "momentum": 1, "nesterov": 2, "adagrad": 3, "rmsprop": 4, "adam": 5}
OPT_STATE = {"sgd": 0, "momentum": 1, "nesterov": 1, "adagrad": 1, "rmsprop": 1, "adam": 2}


def optimizer_update(kind, params, grads, state, t=1, lr=0.01, mu=0.9, rho=0.99, eps=1e-8,
                     beta1=0.9, beta2=0.999):
    """One update of the named optimizer; returns (params', state').
    state: float64[OPT_STATE[kind] * n] (adam: m then v); t: adam timestep (>= 1)."""
    p = _d(params).copy()
    g = _d(grads)
    st = _d(state).copy() if OPT_STATE[kind] else np.zeros(1)
    assert st.size == max(1, OPT_STATE[kind] * p.size)
    lib().oracle_optimizer_update(OPTIMIZERS[kind], p.size, _p(p), _p(g), _p(st), lr, mu, rho, eps,
                                  beta1, beta2, int(t))
    return p, (st if OPT_STATE[kind] else np.zeros(0))


def conv2d_fwd_csr_filter(x, f_row_ptr, f_col_idx, f_val, N, C, H, W, K, R, S, stride=(1, 1), pad=(0, 0),
                          bias=None):
    """Dense input / sparse (CSR, K x C*R*S) filter convolution."""
    P = out_extent(H, pad[0], R, stride[0])
    Q = out_extent(W, pad[1], S, stride[1])
    x = _d(x)
    y = np.empty((N, K * P * Q), dtype=np.float64)
    b = None if bias is None else _d(bias)
    rp, ci, v = _i(f_row_ptr), _i(f_col_idx), _d(f_val)  # kept alive across the call
    assert rp.size == K + 1
    lib().oracle_conv2d_fwd_csr_filter(N, C, H, W, K, R, S, stride[0], stride[1], pad[0], pad[1], _p(x),
                                       _p(rp), _p(ci), _p(v), _p(b), _p(y))
    return y


SPARSITY_THRESHOLD = 0.4  # S:88-92 design decision (the paper gives no threshold)


def decide_format(a, threshold=SPARSITY_THRESHOLD):
    """'sparse' iff nnz / (rows * cols) <= threshold, else 'dense'."""
    a = _d(a)
    nnz = lib().oracle_count_nonzeros(a.size, _p(a))
    return ("sparse" if a.size and nnz / a.size <= threshold else "dense"), int(nnz)


def sgd_update(params, grads, lr=0.01):
    p = _d(params).copy()
    g = _d(grads)
    lib().oracle_sgd_update(p.size, _p(p), _p(g), float(lr))
    return p


# ---- NEXT-4: LeNet-512 + inverted dropout (oracle.c; R22-R24) ----------------

LENET512_HIDDEN = 512


def philox_raw(key0, key1, start, n):
    """Raw 64-bit outputs start..start+n-1 of Philox4x64-10 with key (key0, key1), in
    numpy.random.Philox's output order (oracle_philox_raw)."""
    out = np.empty(n, dtype=np.uint64)
    lib().oracle_philox_raw(int(key0), int(key1), int(start), int(n), _p(out))
    return out


def dropout_mask(seed, step, row0, rows, units, keep_p):
    """uint8 [rows x units] keep mask of global rows row0.. (reading R23)."""
    m = np.empty((rows, units), dtype=np.uint8)
    lib().oracle_dropout_mask(int(seed), int(step), int(row0), int(rows), int(units), float(keep_p), _p(m))
    return m


def dropout_fwd(x, mask, keep_p):
    x = _d(x)
    m = np.ascontiguousarray(mask, dtype=np.uint8)
    assert m.size == x.size
    out = np.empty_like(x)
    lib().oracle_dropout_fwd(x.size, _p(x), _p(m), float(keep_p), _p(out))
    return out


def dropout_bwd(dout, mask, keep_p):
    d = _d(dout)
    m = np.ascontiguousarray(mask, dtype=np.uint8)
    assert m.size == d.size
    dx = np.empty_like(d)
    lib().oracle_dropout_bwd(d.size, _p(d), _p(m), float(keep_p), _p(dx))
    return dx


def lenet512_num_params() -> int:
    return int(lib().oracle_lenet512_num_params())


def lenet512_forward(x, params, train=False, seed=0, step=0, keep_p=1.0, row0=0):
    n = x.shape[0]
    x, prm = _d(x), _d(params)
    H = LENET512_HIDDEN
    a1 = np.empty((n, 6272)); i1 = np.empty((n, 6272), dtype=np.int32)
    a2 = np.empty((n, 3136)); i2 = np.empty((n, 3136), dtype=np.int32)
    z3 = np.empty((n, H)); h = np.empty((n, H)); mask = np.empty((n, H), dtype=np.uint8)
    sc = np.empty((n, 10))
    lib().oracle_lenet512_forward(n, int(row0), _p(x), _p(prm), int(bool(train)), int(seed), int(step),
                                  float(keep_p), _p(a1), _p(i1), _p(a2), _p(i2), _p(z3), _p(h), _p(mask),
                                  _p(sc))
    return dict(a1=a1, i1=i1, a2=a2, i2=i2, z3=z3, h=h, mask=mask, scores=sc)


def lenet512_fwd_bwd(x, labels, params, seed, step, keep_p, n_global=None, row0=0):
    """Returns (grads float64[1663370] pre-scaled by 1/n_global, loss_sum)."""
    n = x.shape[0]
    n_global = n if n_global is None else n_global
    x, lab, prm = _d(x), _i(labels), _d(params)
    g = np.empty(prm.size, dtype=np.float64)
    loss = ctypes.c_double(0.0)
    lib().oracle_lenet512_fwd_bwd(n, int(n_global), int(row0), _p(x), _p(lab), _p(prm), int(seed), int(step),
                                  float(keep_p), _p(g),
                                  ctypes.cast(ctypes.pointer(loss), ctypes.POINTER(ctypes.c_double)))
    return g, loss.value


def lenet512_predict(x, params):
    n = x.shape[0]
    x, prm = _d(x), _d(params)
    pred = np.empty(n, dtype=np.int32)
    probs = np.empty((n, 10), dtype=np.float64)
    lib().oracle_lenet512_predict(n, _p(x), _p(prm), _p(pred), _p(probs))
    return pred, probs
