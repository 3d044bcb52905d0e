"""Python binding of libsysml.so -- the B200-native conv2d-family hot path of
arXiv 1802.04647 ("Deep Learning with Apache SystemML", §3 GPU backend).

Argument marshalling only: every step of the path runs in the CUDA kernels of
``csrc/`` behind the C ABI declared in ``include/sysml.h``; the names below are
that ABI's names.  PyTorch supplies device memory, streams and process groups.
There is no CPU fallback: importing works anywhere (so the symbol table can be
checked on a CPU box), but every compute call requires CUDA tensors and raises
if the library or a GPU is missing.

Tensor encoding (§3 "Tensor Representation"): [N, C, H, W] is the
row-major matrix N x (C*H*W); tensors passed here are 2-D float32 CUDA tensors
of that shape (any contiguous shape with the right numel is accepted).
"""
from __future__ import annotations

import ctypes
import threading
import os
from dataclasses import dataclass
from typing import Optional

from . import _build

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libsysml.so")

MATH_FP32 = 0
MATH_TF32 = 1
_MATH = {"fp32": MATH_FP32, "tf32": MATH_TF32, MATH_FP32: MATH_FP32, MATH_TF32: MATH_TF32}

STATUS = {0: "SYSML_OK", 1: "SYSML_ERR_ARG", 2: "SYSML_ERR_SHAPE", 3: "SYSML_ERR_UNSUPPORTED",
          4: "SYSML_ERR_CUDA", 5: "SYSML_ERR_NCCL", 6: "SYSML_ERR_WORKSPACE"}

# every symbol include/sysml.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "sysml_version", "sysml_last_error", "sysml_last_route", "sysml_device_sm_count", "sysml_launch_counter",
    "sysml_conv2d_workspace_size", "sysml_conv2d",
    "sysml_conv2d_bwd_filter_workspace_size", "sysml_conv2d_bwd_filter",
    "sysml_conv2d_bwd_data_workspace_size", "sysml_conv2d_bwd_data",
    "sysml_bias_add", "sysml_relu_maxpool", "sysml_maxpool_bwd",
    "sysml_conv2d_bias_relu_maxpool_workspace_size", "sysml_conv2d_bias_relu_maxpool",
    "sysml_csr_check",
    "sysml_lenet_num_params", "sysml_lenet_create", "sysml_lenet_destroy", "sysml_lenet_fwd_bwd",
    "sysml_sgd_update", "sysml_lenet_step", "sysml_lenet_step_host",
    "sysml_lenet_set_timing", "sysml_lenet_get_timing",
    "sysml_optimizer_state_floats", "sysml_optimizer_update", "sysml_lenet_step_opt",
    "sysml_lenet_step_host_pipelined", "sysml_decide_format",
    "sysml_lenet512_num_params", "sysml_lenet512_create", "sysml_lenet_set_dropout",
    "sysml_lenet_get_dropout_step", "sysml_lenet_handle_num_params", "sysml_affine",
    "sysml_conv2d_multi_workspace_size", "sysml_conv2d_multi", "sysml_conv2d_multi_bwd_data",
    "sysml_conv2d_multi_bwd_filter",
    "sysml_conv2d_csr_filter", "sysml_count_nonzeros", "sysml_dense_to_csr", "sysml_lenet_predict",
)


class SysmlError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class ConvDesc(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in
                ("N", "C", "H", "W", "K", "R", "S", "stride_h", "stride_w", "pad_h", "pad_w", "math")]

    @property
    def P(self):
        return (self.H + 2 * self.pad_h - self.R) // self.stride_h + 1

    @property
    def Q(self):
        return (self.W + 2 * self.pad_w - self.S) // self.stride_w + 1


class PoolDesc(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in
                ("N", "C", "H", "W", "R", "S", "stride_h", "stride_w", "pad_h", "pad_w", "relu")]

    @property
    def P(self):
        return (self.H + 2 * self.pad_h - self.R) // self.stride_h + 1

    @property
    def Q(self):
        return (self.W + 2 * self.pad_w - self.S) // self.stride_w + 1


class OptimizerDesc(ctypes.Structure):
    """sysml_optimizer_desc (include/sysml.h): the six NN-library optimizers."""
    _fields_ = [("kind", ctypes.c_int32), ("lr", ctypes.c_float), ("mu", ctypes.c_float),
                ("rho", ctypes.c_float), ("eps", ctypes.c_float), ("beta1", ctypes.c_float),
                ("beta2", ctypes.c_float)]


OPTIMIZERS = {"sgd": 0, "momentum": 1, "nesterov": 2, "adagrad": 3, "rmsprop": 4, "adam": 5}


def optimizer_desc(kind, lr=0.01, mu=0.9, rho=0.99, eps=1e-8, beta1=0.9, beta2=0.999) -> OptimizerDesc:
    """Defaults: S:285 (eps 1e-8, mu 0.9, rho 0.99, beta1 0.9, beta2 0.999) and lr 0.01."""
    return OptimizerDesc(OPTIMIZERS[kind], lr, mu, rho, eps, beta1, beta2)


class _Csr(ctypes.Structure):
    _fields_ = [("rows", ctypes.c_int64), ("cols", ctypes.c_int64), ("nnz", ctypes.c_int64),
                ("row_ptr", ctypes.c_void_p), ("col_idx", ctypes.c_void_p), ("val", ctypes.c_void_p)]


class _Input(ctypes.Structure):
    _fields_ = [("is_csr", ctypes.c_int32), ("dense", ctypes.c_void_p), ("csr", _Csr)]


@dataclass
class CSR:
    """Device CSR matrix (§3 "Sparse Operations"): int32 row_ptr[rows+1],
    int32 col_idx[nnz], float32 val[nnz] (torch CUDA tensors)."""
    row_ptr: "object"
    col_idx: "object"
    val: "object"
    rows: int
    cols: int

    @property
    def nnz(self):
        return int(self.col_idx.numel())


def conv_desc(N, C, H, W, K, R, S, stride=(1, 1), pad=(0, 0), math="tf32") -> ConvDesc:
    stride = (stride, stride) if isinstance(stride, int) else tuple(stride)
    pad = (pad, pad) if isinstance(pad, int) else tuple(pad)
    return ConvDesc(N, C, H, W, K, R, S, stride[0], stride[1], pad[0], pad[1], _MATH[math])


def pool_desc(N, C, H, W, R, S, stride=None, pad=(0, 0), relu=True) -> PoolDesc:
    stride = (R, S) if stride is None else ((stride, stride) if isinstance(stride, int) else tuple(stride))
    pad = (pad, pad) if isinstance(pad, int) else tuple(pad)
    return PoolDesc(N, C, H, W, R, S, stride[0], stride[1], pad[0], pad[1], int(bool(relu)))


_lib = None


def lib(build_if_missing: bool = False):
    """Load libsysml.so (raises if absent: no fallback path exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if build_if_missing and not os.path.exists(LIB_PATH):
        _build.build()
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libsysml.so not built ({LIB_PATH}); run __graft_entry__.build()")
    L = ctypes.CDLL(LIB_PATH)
    c_i32, c_i64, vp, sz = ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p, ctypes.c_size_t
    CD, PD, IN, CS = ctypes.POINTER(ConvDesc), ctypes.POINTER(PoolDesc), ctypes.POINTER(_Input), ctypes.POINTER(_Csr)
    psz = ctypes.POINTER(ctypes.c_size_t)
    sig = {
        "sysml_version": (ctypes.c_char_p, []),
        "sysml_last_error": (ctypes.c_char_p, []),
        "sysml_last_route": (ctypes.c_char_p, []),
        "sysml_device_sm_count": (c_i32, []),
        "sysml_launch_counter": (c_i64, []),
        "sysml_conv2d_workspace_size": (c_i32, [CD, c_i32, psz]),
        "sysml_conv2d": (c_i32, [CD, IN, vp, vp, vp, vp, sz, vp]),
        "sysml_conv2d_bwd_filter_workspace_size": (c_i32, [CD, c_i32, psz]),
        "sysml_conv2d_bwd_filter": (c_i32, [CD, IN, vp, vp, vp, vp, sz, vp]),
        "sysml_conv2d_bwd_data_workspace_size": (c_i32, [CD, psz]),
        "sysml_conv2d_bwd_data": (c_i32, [CD, vp, vp, vp, vp, sz, vp]),
        "sysml_bias_add": (c_i32, [c_i32, c_i32, c_i32, vp, vp, vp]),
        "sysml_relu_maxpool": (c_i32, [PD, vp, vp, vp, vp]),
        "sysml_maxpool_bwd": (c_i32, [PD, vp, vp, vp, vp, vp]),
        "sysml_conv2d_bias_relu_maxpool_workspace_size": (c_i32, [CD, PD, c_i32, psz]),
        "sysml_conv2d_bias_relu_maxpool": (c_i32, [CD, PD, IN, vp, vp, vp, vp, vp, sz, vp]),
        "sysml_csr_check": (c_i32, [CS, ctypes.POINTER(c_i64), vp]),
        "sysml_lenet_num_params": (c_i64, []),
        "sysml_lenet_create": (c_i32, [c_i32, c_i32, c_i32, c_i64, ctypes.POINTER(vp)]),
        "sysml_lenet_destroy": (c_i32, [vp]),
        "sysml_lenet_fwd_bwd": (c_i32, [vp, vp, IN, vp, c_i32, c_i64, vp, vp, vp]),
        "sysml_sgd_update": (c_i32, [vp, vp, c_i64, ctypes.c_float, vp]),
        "sysml_lenet_step": (c_i32, [vp, vp, vp, IN, vp, c_i32, c_i64, ctypes.c_float, vp, vp, vp]),
        "sysml_lenet_step_host": (c_i32, [vp, vp, vp, vp, vp, c_i32, c_i64, ctypes.c_float, vp, vp, vp]),
        "sysml_lenet_set_timing": (c_i32, [vp, c_i32]),
        "sysml_optimizer_state_floats": (c_i32, [c_i32]),
        "sysml_conv2d_csr_filter": (c_i32, [CD, IN, CS, vp, vp, vp]),
        "sysml_lenet_predict": (c_i32, [vp, vp, IN, c_i32, vp, vp, vp]),
        "sysml_count_nonzeros": (c_i32, [vp, c_i64, ctypes.POINTER(c_i64), vp]),
        "sysml_dense_to_csr": (c_i32, [vp, c_i64, c_i64, vp, vp, vp, vp]),
        "sysml_decide_format": (c_i32, [vp, c_i64, ctypes.c_double, ctypes.POINTER(c_i32),
                                        ctypes.POINTER(c_i64), vp]),
        "sysml_lenet_step_host_pipelined": (c_i32, [vp, vp, vp, vp, vp, c_i32, vp, vp, c_i32, c_i64,
                                                    ctypes.c_float, vp, vp, vp]),
        "sysml_optimizer_update": (c_i32, [ctypes.POINTER(OptimizerDesc), vp, vp, vp, c_i64, c_i64, vp]),
        "sysml_lenet_step_opt": (c_i32, [vp, vp, vp, vp, ctypes.POINTER(OptimizerDesc), c_i64, IN, vp, c_i32,
                                         c_i64, vp, vp, vp]),
        "sysml_lenet_get_timing": (c_i32, [vp, c_i32, ctypes.POINTER(c_i32), ctypes.POINTER(ctypes.c_double),
                                           ctypes.POINTER(c_i64), ctypes.POINTER(ctypes.c_char_p)]),
        "sysml_lenet512_num_params": (c_i64, []),
        "sysml_lenet512_create": (c_i32, [c_i32, c_i32, c_i32, c_i64, ctypes.c_float, ctypes.c_uint64,
                                          ctypes.POINTER(vp)]),
        "sysml_lenet_set_dropout": (c_i32, [vp, c_i64, c_i64, vp]),
        "sysml_lenet_get_dropout_step": (c_i32, [vp, ctypes.POINTER(c_i64)]),
        "sysml_lenet_handle_num_params": (c_i64, [vp]),
        "sysml_affine": (c_i32, [c_i32, c_i32, c_i32, vp, vp, vp, c_i32, c_i32, vp, vp]),
        "sysml_conv2d_multi_workspace_size": (c_i32, [CD, c_i32, vp, c_i32, c_i32, psz]),
        "sysml_conv2d_multi": (c_i32, [CD, c_i32, vp, IN, vp, vp, vp, vp, sz, vp]),
        "sysml_conv2d_multi_bwd_data": (c_i32, [CD, c_i32, vp, vp, vp, vp, vp, sz, vp]),
        "sysml_conv2d_multi_bwd_filter": (c_i32, [CD, c_i32, vp, IN, vp, vp, vp, vp, sz, vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype, fn.argtypes = res, args
    _lib = L
    return L


def _check(status: int):
    if status != 0:
        raise SysmlError(status, lib().sysml_last_error().decode())


# ---------------------------------------------------------------------------- helpers
def _torch():
    import torch
    return torch


def _stream(stream=None):
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _ptr(t, dtype=None, name="tensor"):
    if t is None:
        return None
    torch = _torch()
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA torch.Tensor (no CPU path exists)")
    if dtype is not None and t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


def _input(x) -> _Input:
    torch = _torch()
    if isinstance(x, CSR):
        return _Input(1, None, _Csr(x.rows, x.cols, x.nnz,
                                    _ptr(x.row_ptr, torch.int32, "row_ptr").value,
                                    _ptr(x.col_idx, torch.int32, "col_idx").value if x.nnz else None,
                                    _ptr(x.val, torch.float32, "val").value if x.nnz else None))
    return _Input(0, _ptr(x, torch.float32, "x").value, _Csr())


_ws_keep = threading.local()


def _workspace(nbytes: int, workspace=None, stream=None):
    """The caller's workspace if large enough, else a fresh buffer allocated on the stream the
    kernel runs on (so the caching allocator orders its reuse after that kernel), kept alive
    per thread and stream until the next call on them."""
    torch = _torch()
    if nbytes == 0:
        return None, 0
    if workspace is not None and workspace.numel() * workspace.element_size() >= nbytes:
        return ctypes.c_void_p(workspace.data_ptr()), workspace.numel() * workspace.element_size()
    s = stream if stream is not None else torch.cuda.current_stream()
    with torch.cuda.stream(s):
        buf = torch.empty(nbytes, dtype=torch.uint8, device=s.device)
    keep = getattr(_ws_keep, "bufs", None)
    if keep is None:
        keep = _ws_keep.bufs = {}
    keep[(s.device.index, s.cuda_stream)] = buf
    return ctypes.c_void_p(buf.data_ptr()), nbytes


def _ws_size(fn, *args) -> int:
    n = ctypes.c_size_t(0)
    _check(fn(*args, ctypes.byref(n)))
    return n.value


# ---------------------------------------------------------------------------- operators
def sysml_conv2d(x, f, d: ConvDesc, bias=None, out=None, workspace=None, stream=None):
    """conv2d / conv2d_bias_add (§3 Builtin NN Functions): N x (K*P*Q)."""
    torch = _torch()
    L = lib()
    inp = _input(x)
    if out is None:
        out = torch.empty((d.N, d.K * d.P * d.Q), dtype=torch.float32, device="cuda")
    nb = _ws_size(L.sysml_conv2d_workspace_size, ctypes.byref(d), inp.is_csr)
    ws, wsb = _workspace(nb, workspace, stream)
    _check(L.sysml_conv2d(ctypes.byref(d), ctypes.byref(inp), _ptr(f, torch.float32, "f"),
                          _ptr(bias, torch.float32, "bias"), _ptr(out, torch.float32, "out"),
                          ws, wsb, _stream(stream)))
    return out


def sysml_conv2d_bwd_filter(x, dy, d: ConvDesc, df=None, db=None, want_db=True, workspace=None, stream=None):
    torch = _torch()
    L = lib()
    inp = _input(x)
    if df is None:
        df = torch.empty((d.K, d.C * d.R * d.S), dtype=torch.float32, device="cuda")
    if db is None and want_db:
        db = torch.empty((d.K,), dtype=torch.float32, device="cuda")
    nb = _ws_size(L.sysml_conv2d_bwd_filter_workspace_size, ctypes.byref(d), inp.is_csr)
    ws, wsb = _workspace(nb, workspace, stream)
    _check(L.sysml_conv2d_bwd_filter(ctypes.byref(d), ctypes.byref(inp), _ptr(dy, torch.float32, "dy"),
                                     _ptr(df, torch.float32, "df"), _ptr(db, torch.float32, "db"),
                                     ws, wsb, _stream(stream)))
    return df, db


def sysml_conv2d_bwd_data(f, dy, d: ConvDesc, dx=None, workspace=None, stream=None):
    torch = _torch()
    L = lib()
    if dx is None:
        dx = torch.empty((d.N, d.C * d.H * d.W), dtype=torch.float32, device="cuda")
    nb = _ws_size(L.sysml_conv2d_bwd_data_workspace_size, ctypes.byref(d))
    ws, wsb = _workspace(nb, workspace, stream)
    _check(L.sysml_conv2d_bwd_data(ctypes.byref(d), _ptr(f, torch.float32, "f"), _ptr(dy, torch.float32, "dy"),
                                   _ptr(dx, torch.float32, "dx"), ws, wsb, _stream(stream)))
    return dx


def _ptr_array(ts, torch, what):
    arr = (ctypes.c_void_p * len(ts))()
    for i, t in enumerate(ts):
        arr[i] = _ptr(t, torch.float32, f"{what}[{i}]") if t is not None else None
    return arr


def _multi_setup(d: ConvDesc, ks, op, is_csr, workspace, stream):
    L = lib()
    kc = (ctypes.c_int32 * len(ks))(*[int(k) for k in ks])
    nb = ctypes.c_size_t(0)
    _check(L.sysml_conv2d_multi_workspace_size(ctypes.byref(d), len(ks), kc, op, int(is_csr), ctypes.byref(nb)))
    ws, wsb = _workspace(nb.value, workspace, stream)
    return L, kc, ws, wsb


def sysml_conv2d_multi(x, fs, d: ConvDesc, biases=None, out=None, workspace=None, stream=None):
    """Horizontal fusion: the convs with filter banks fs (k_i x CRS) over the shared
    input x, as one conv; returns y_cat N x (sum k_i * P * Q) (channel concatenation)."""
    torch = _torch()
    ks = [f.shape[0] for f in fs]
    inp = _input(x)
    if out is None:
        out = torch.empty((d.N, d.K * d.P * d.Q), dtype=torch.float32, device="cuda")
    L, kc, ws, wsb = _multi_setup(d, ks, 0, isinstance(x, CSR), workspace, stream)
    fa = _ptr_array(fs, torch, "f")
    ba = _ptr_array(biases, torch, "bias") if biases is not None else None
    _check(L.sysml_conv2d_multi(ctypes.byref(d), len(ks), kc, ctypes.byref(inp), fa, ba,
                                _ptr(out, torch.float32, "y_cat"), ws, wsb, _stream(stream)))
    return out


def sysml_conv2d_multi_bwd_data(fs, dy_cat, d: ConvDesc, dx=None, workspace=None, stream=None):
    """sum_i conv2d_bwd_data(fs[i], dy_i) in one kernel (dy_cat: channel concatenation)."""
    torch = _torch()
    ks = [f.shape[0] for f in fs]
    if dx is None:
        dx = torch.empty((d.N, d.C * d.H * d.W), dtype=torch.float32, device="cuda")
    L, kc, ws, wsb = _multi_setup(d, ks, 1, False, workspace, stream)
    _check(L.sysml_conv2d_multi_bwd_data(ctypes.byref(d), len(ks), kc, _ptr_array(fs, torch, "f"),
                                         _ptr(dy_cat, torch.float32, "dy_cat"), _ptr(dx, torch.float32, "dx"),
                                         ws, wsb, _stream(stream)))
    return dx


def sysml_conv2d_multi_bwd_filter(x, dy_cat, d: ConvDesc, ks, want_db=True, workspace=None, stream=None):
    """Per-op (df_i, db_i) of the horizontally fused convs from x and dy_cat."""
    torch = _torch()
    inp = _input(x)
    crs = d.C * d.R * d.S
    dfs = [torch.empty((k, crs), dtype=torch.float32, device="cuda") for k in ks]
    dbs = [torch.empty((k,), dtype=torch.float32, device="cuda") for k in ks] if want_db else None
    L, kc, ws, wsb = _multi_setup(d, ks, 2, isinstance(x, CSR), workspace, stream)
    _check(L.sysml_conv2d_multi_bwd_filter(ctypes.byref(d), len(ks), kc, ctypes.byref(inp),
                                           _ptr(dy_cat, torch.float32, "dy_cat"), _ptr_array(dfs, torch, "df"),
                                           _ptr_array(dbs, torch, "db") if want_db else None, ws, wsb,
                                           _stream(stream)))
    return dfs, dbs


def sysml_affine(x, W, b=None, relu=False, math="tf32", out=None, stream=None):
    """Affine layer forward (sysml_affine): out = x W^T + b (relu optional); x M x K, W N x K."""
    torch = _torch()
    M, K = x.shape
    N = W.shape[0]
    if out is None:
        out = torch.empty((M, N), dtype=torch.float32, device="cuda")
    _check(lib().sysml_affine(int(M), int(N), int(K), _ptr(x, torch.float32, "x"), _ptr(W, torch.float32, "W"),
                              _ptr(b, torch.float32, "b"), int(bool(relu)), _MATH[math],
                              _ptr(out, torch.float32, "out"), _stream(stream)))
    return out


def sysml_bias_add(y, bias, N, K, PQ, stream=None):
    torch = _torch()
    _check(lib().sysml_bias_add(N, K, PQ, _ptr(y, torch.float32, "y"), _ptr(bias, torch.float32, "bias"),
                                _stream(stream)))
    return y


def sysml_relu_maxpool(x, d: PoolDesc, out=None, argmax=None, want_argmax=True, stream=None):
    torch = _torch()
    if out is None:
        out = torch.empty((d.N, d.C * d.P * d.Q), dtype=torch.float32, device="cuda")
    if argmax is None and want_argmax:
        argmax = torch.empty((d.N, d.C * d.P * d.Q), dtype=torch.int32, device="cuda")
    _check(lib().sysml_relu_maxpool(ctypes.byref(d), _ptr(x, torch.float32, "x"), _ptr(out, torch.float32, "out"),
                                    _ptr(argmax, torch.int32, "argmax"), _stream(stream)))
    return out, argmax


def sysml_maxpool_bwd(argmax, dout, d: PoolDesc, out_mask=None, dx=None, stream=None):
    torch = _torch()
    if dx is None:
        dx = torch.empty((d.N, d.C * d.H * d.W), dtype=torch.float32, device="cuda")
    _check(lib().sysml_maxpool_bwd(ctypes.byref(d), _ptr(argmax, torch.int32, "argmax"),
                                   _ptr(dout, torch.float32, "dout"), _ptr(out_mask, torch.float32, "out_mask"),
                                   _ptr(dx, torch.float32, "dx"), _stream(stream)))
    return dx


def sysml_conv2d_bias_relu_maxpool(x, f, bias, cd: ConvDesc, pd: PoolDesc, out=None, argmax=None,
                                   workspace=None, stream=None):
    torch = _torch()
    L = lib()
    inp = _input(x)
    if out is None:
        out = torch.empty((pd.N, pd.C * pd.P * pd.Q), dtype=torch.float32, device="cuda")
    if argmax is None:
        argmax = torch.empty((pd.N, pd.C * pd.P * pd.Q), dtype=torch.int32, device="cuda")
    nb = _ws_size(L.sysml_conv2d_bias_relu_maxpool_workspace_size, ctypes.byref(cd), ctypes.byref(pd), inp.is_csr)
    ws, wsb = _workspace(nb, workspace, stream)
    _check(L.sysml_conv2d_bias_relu_maxpool(ctypes.byref(cd), ctypes.byref(pd), ctypes.byref(inp),
                                            _ptr(f, torch.float32, "f"), _ptr(bias, torch.float32, "bias"),
                                            _ptr(out, torch.float32, "out"), _ptr(argmax, torch.int32, "argmax"),
                                            ws, wsb, _stream(stream)))
    return out, argmax


def sysml_csr_check(m: CSR, stream=None) -> int:
    torch = _torch()
    v = ctypes.c_int64(0)
    c = _Csr(m.rows, m.cols, m.nnz, _ptr(m.row_ptr, torch.int32).value,
             _ptr(m.col_idx, torch.int32).value if m.nnz else None,
             _ptr(m.val, torch.float32).value if m.nnz else None)
    _check(lib().sysml_csr_check(ctypes.byref(c), ctypes.byref(v), _stream(stream)))
    return v.value


def sysml_sgd_update(params, grads, lr=0.01, stream=None):
    torch = _torch()
    _check(lib().sysml_sgd_update(_ptr(params, torch.float32, "params"), _ptr(grads, torch.float32, "grads"),
                                  params.numel(), ctypes.c_float(lr), _stream(stream)))
    return params


def _csr_struct(m):
    torch = _torch()
    return _Csr(m.rows, m.cols, m.nnz, _ptr(m.row_ptr, torch.int32).value,
                _ptr(m.col_idx, torch.int32).value if m.nnz else None, _ptr(m.val, torch.float32).value if m.nnz else None)


def sysml_conv2d_csr_filter(x, f: "CSR", d, bias=None, out=None, stream=None):
    """Convolution with a CSR filter bank (K x C*R*S): dense input / sparse filter, or sparse /
    sparse when x is a CSR."""
    torch = _torch()
    y = out if out is not None else torch.empty(d.N, d.K * d.P * d.Q, device="cuda", dtype=torch.float32)
    inp = _input(x)
    fc = _csr_struct(f)
    _check(lib().sysml_conv2d_csr_filter(ctypes.byref(d), ctypes.byref(inp), ctypes.byref(fc),
                                         _ptr(bias, torch.float32, "bias"), _ptr(y, torch.float32, "y"), _stream(stream)))
    return y


SPARSITY_THRESHOLD = 0.4


def sysml_count_nonzeros(x, stream=None) -> int:
    torch = _torch()
    n = ctypes.c_int64(0)
    _check(lib().sysml_count_nonzeros(_ptr(x, torch.float32, "x"), x.numel(), ctypes.byref(n), _stream(stream)))
    return n.value


def dense_to_csr(x, stream=None) -> "CSR":
    """GPU dense (rows x cols, fp32) -> CSR, columns ascending per row (sysml_dense_to_csr)."""
    torch = _torch()
    rows, cols = x.shape
    nnz = sysml_count_nonzeros(x, stream)
    rp = torch.empty(rows + 1, device="cuda", dtype=torch.int32)
    ci = torch.empty(max(nnz, 1), device="cuda", dtype=torch.int32)
    v = torch.empty(max(nnz, 1), device="cuda", dtype=torch.float32)
    _check(lib().sysml_dense_to_csr(_ptr(x, torch.float32, "x"), rows, cols, _ptr(rp), _ptr(ci), _ptr(v), _stream(stream)))
    return CSR(rp, ci[:nnz], v[:nnz], rows, cols)


def decide_format(x, threshold=SPARSITY_THRESHOLD, stream=None):
    """P:163-165 / S:88-96: the CSR form of x if nnz / (rows*cols) <= threshold, else x itself
    (the rule is sysml_decide_format in the C ABI)."""
    torch = _torch()
    sparse = ctypes.c_int32(0)
    nnz = ctypes.c_int64(0)
    _check(lib().sysml_decide_format(_ptr(x, torch.float32, "x"), x.numel(), float(threshold),
                                     ctypes.byref(sparse), ctypes.byref(nnz), _stream(stream)))
    return dense_to_csr(x, stream) if sparse.value else x


def sysml_optimizer_update(desc, params, grads, state, t=1, stream=None):
    """One in-place optimizer update (sysml_optimizer_update)."""
    torch = _torch()
    _check(lib().sysml_optimizer_update(ctypes.byref(desc), _ptr(params, torch.float32, "params"),
                                        _ptr(grads, torch.float32, "grads"), _ptr(state, torch.float32, "state"),
                                        params.numel(), int(t), _stream(stream)))
    return params


def sysml_last_route() -> str:
    """The kernels the last conv call on this thread launched (sysml_last_route)."""
    return lib().sysml_last_route().decode()


def sysml_launch_counter() -> int:
    return int(lib().sysml_launch_counter())


def sysml_version() -> str:
    return lib().sysml_version().decode()


def nccl_comm_ptr(group=None, allow_single: bool = False) -> Optional[int]:
    """ncclComm_t of torch's ProcessGroupNCCL (created lazily; run one collective first).
    None for a single rank unless allow_single (tests of the in-library allreduce path)."""
    torch = _torch()
    import torch.distributed as dist
    if not dist.is_initialized() or (dist.get_world_size() == 1 and not allow_single):
        return None
    pg = group or dist.distributed_c10d._get_default_group()
    be = pg._get_backend(torch.device("cuda"))
    return int(be._comm_ptr())


class LeNet:
    """Minibatch SGD-step driver (Listing 1; P:142 LeNet; P:187-192 data-parallel plan).

    model="lenet-min" (default): conv-relu-pool x2, affine 3136->10 (83,466 parameters).
    model="lenet512": SystemML's mnist_lenet topology with affine 3136->512, relu, inverted
    dropout (keep_p, Philox mask stream ``seed``), affine 512->10 (1,663,370 parameters;
    sysml_lenet512_create, NEXT-4)."""

    NUM_PARAMS = 83466
    NUM_PARAMS_512 = 1663370

    def __init__(self, max_local_batch: int, math="tf32", csr=False, max_nnz=0, model="lenet-min",
                 keep_p=0.5, seed=0):
        L = lib()
        h = ctypes.c_void_p()
        if model == "lenet-min":
            _check(L.sysml_lenet_create(int(max_local_batch), _MATH[math], int(bool(csr)), int(max_nnz),
                                        ctypes.byref(h)))
        elif model == "lenet512":
            _check(L.sysml_lenet512_create(int(max_local_batch), _MATH[math], int(bool(csr)), int(max_nnz),
                                           ctypes.c_float(keep_p), ctypes.c_uint64(int(seed)), ctypes.byref(h)))
        else:
            raise ValueError(f"unknown model {model!r}")
        self.h = h
        self.model = model
        self.num_params = int(L.sysml_lenet_handle_num_params(h))
        self.max_local_batch = max_local_batch
        self.csr = bool(csr)

    def set_dropout(self, row0=0, step=0, stream=None):
        """LeNet-512: global row offset of the local shard and the device mask-step counter."""
        _check(lib().sysml_lenet_set_dropout(self.h, int(row0), int(step), _stream(stream)))

    def dropout_step(self) -> int:
        v = ctypes.c_int64(0)
        _check(lib().sysml_lenet_get_dropout_step(self.h, ctypes.byref(v)))
        return v.value

    def close(self):
        if getattr(self, "h", None):
            lib().sysml_lenet_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def fwd_bwd(self, params, x, labels, n_global, grads, loss_sum=None, stream=None):
        torch = _torch()
        inp = _input(x)
        n = x.rows if isinstance(x, CSR) else x.shape[0]
        _check(lib().sysml_lenet_fwd_bwd(self.h, _ptr(params, torch.float32, "params"), ctypes.byref(inp),
                                         _ptr(labels, torch.int32, "labels"), int(n), int(n_global),
                                         _ptr(grads, torch.float32, "grads"), _ptr(loss_sum, torch.float32, "loss_sum"),
                                         _stream(stream)))

    def predict(self, params, x, probs=False, stream=None):
        """Scoring (sysml_lenet_predict): predicted labels (int32[n]) and, if probs, the softmax
        probabilities (fp32[n, 10])."""
        torch = _torch()
        inp = _input(x)
        n = x.rows if isinstance(x, CSR) else x.shape[0]
        pred = torch.empty(n, device="cuda", dtype=torch.int32)
        pr = torch.empty(n, 10, device="cuda", dtype=torch.float32) if probs else None
        _check(lib().sysml_lenet_predict(self.h, _ptr(params, torch.float32, "params"), ctypes.byref(inp), int(n),
                                         _ptr(pred), _ptr(pr), _stream(stream)))
        return (pred, pr) if probs else pred

    def step(self, params, grads, x, labels, n_global, lr=0.01, nccl_comm=None, loss_sum=None, stream=None):
        torch = _torch()
        inp = _input(x)
        n = x.rows if isinstance(x, CSR) else x.shape[0]
        _check(lib().sysml_lenet_step(self.h, _ptr(params, torch.float32, "params"), _ptr(grads, torch.float32, "grads"),
                                      ctypes.byref(inp), _ptr(labels, torch.int32, "labels"), int(n), int(n_global),
                                      ctypes.c_float(lr), ctypes.c_void_p(nccl_comm) if nccl_comm else None,
                                      _ptr(loss_sum, torch.float32, "loss_sum"), _stream(stream)))

    def step_opt(self, params, grads, state, desc, t, x, labels, n_global, nccl_comm=None, loss_sum=None,
                 stream=None):
        """One step with any of the six optimizers (sysml_lenet_step_opt); state: device fp32
        [sysml_optimizer_state_floats(kind) * 83466] (None for SGD), t: adam timestep >= 1."""
        torch = _torch()
        inp = _input(x)
        n = x.rows if isinstance(x, CSR) else x.shape[0]
        _check(lib().sysml_lenet_step_opt(self.h, _ptr(params, torch.float32, "params"), _ptr(grads, torch.float32, "grads"),
                                          _ptr(state, torch.float32, "state"), ctypes.byref(desc), int(t),
                                          ctypes.byref(inp), _ptr(labels, torch.int32, "labels"), int(n), int(n_global),
                                          ctypes.c_void_p(nccl_comm) if nccl_comm else None,
                                          _ptr(loss_sum, torch.float32, "loss_sum"), _stream(stream)))

    def step_host(self, params, grads, x_host, labels_host, n_global, lr=0.01, nccl_comm=None, stream=None) -> float:
        """End-to-end step from HOST (ideally pinned) float32 / int32 CPU tensors."""
        torch = _torch()
        loss = ctypes.c_float(0.0)
        if x_host.is_cuda or labels_host.is_cuda or x_host.dtype != torch.float32 or labels_host.dtype != torch.int32:
            raise TypeError("step_host takes float32 / int32 CPU tensors")
        _check(lib().sysml_lenet_step_host(self.h, _ptr(params, torch.float32), _ptr(grads, torch.float32),
                                           ctypes.c_void_p(x_host.data_ptr()), ctypes.c_void_p(labels_host.data_ptr()),
                                           int(x_host.shape[0]), int(n_global), ctypes.c_float(lr),
                                           ctypes.c_void_p(nccl_comm) if nccl_comm else None,
                                           ctypes.byref(loss), _stream(stream)))
        return loss.value

    def step_host_pipelined(self, params, grads, x_host, labels_host, n_global, next_x=None, next_labels=None,
                            lr=0.01, nccl_comm=None, stream=None) -> float:
        """step_host for a loop over host batches: the next batch (pinned, unchanged until the
        next call) is copied to the device while this step computes
        (sysml_lenet_step_host_pipelined)."""
        torch = _torch()
        loss = ctypes.c_float(0.0)
        for t in (x_host, labels_host) + ((next_x, next_labels) if next_x is not None else ()):
            if t.is_cuda:
                raise TypeError("step_host_pipelined takes CPU (pinned) tensors")
        if x_host.dtype != torch.float32 or labels_host.dtype != torch.int32:
            raise TypeError("step_host_pipelined takes float32 / int32 CPU tensors")
        nxt = next_x is not None
        _check(lib().sysml_lenet_step_host_pipelined(
            self.h, _ptr(params, torch.float32), _ptr(grads, torch.float32),
            ctypes.c_void_p(x_host.data_ptr()), ctypes.c_void_p(labels_host.data_ptr()), int(x_host.shape[0]),
            ctypes.c_void_p(next_x.data_ptr()) if nxt else None,
            ctypes.c_void_p(next_labels.data_ptr()) if nxt else None, int(next_x.shape[0]) if nxt else 0,
            int(n_global), ctypes.c_float(lr), ctypes.c_void_p(nccl_comm) if nccl_comm else None,
            ctypes.byref(loss), _stream(stream)))
        return loss.value

    def set_timing(self, enable: bool):
        _check(lib().sysml_lenet_set_timing(self.h, int(bool(enable))))

    def get_timing(self, reset=False):
        n = 16
        ms = (ctypes.c_double * n)()
        calls = (ctypes.c_int64 * n)()
        names = (ctypes.c_char_p * n)()
        ns = ctypes.c_int32(0)
        _check(lib().sysml_lenet_get_timing(self.h, n, ctypes.byref(ns), ms, calls, names))
        out = {names[i].decode(): (ms[i], calls[i]) for i in range(ns.value)}
        if reset:
            _check(lib().sysml_lenet_get_timing(self.h, -1, None, None, None, None))
        return out
