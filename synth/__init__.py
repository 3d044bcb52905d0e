"""Seeded synthetic input generators shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method (no convolution, pooling, loss or
update).  It only draws numbers and encodes them (dense row-major N x (C*H*W),
or CSR), so that the fp64 oracle (``oracle/``) and the CUDA library
(``paper_1802_04647_b200``) can be fed bit-identical inputs without sharing any
code.  The recipe is the one stated in DESIGN.md "Input recipe" (after SURVEY.md
§8(d) "Input generators"):

* every generator takes an explicit ``seed`` list; numbers come from NumPy
  PCG64 ``default_rng([180204647, *seed])``;
* family **U** (continuous):  X ~ U(-1,1), F ~ N(0, 2/(C R S)), b ~ N(0, 0.1^2),
  dY ~ N(0,1), labels ~ U{0..9};
* family **M** (MNIST-shaped, §1 "sparse/ultra-sparse inputs", BJ cfg 3):
  1x28x28, non-zeros only in the central 20x20 box, per image Bernoulli(p_i),
  p_i ~ U(0.25, 0.50) (mean density 0.191), values k/255, k ~ U{1..255};
* family **G** (dyadic grid): every value has <= 11 significant bits so it is
  exact in TF32 and every partial sum of the conv is exact in fp32;
* LeNet parameters: Glorot-uniform (SPEC.md nn-layers DESIGN DECISIONS) with a
  fixed seed.

All arrays are float32 (int32 for indices/labels), C-contiguous.
"""
from __future__ import annotations

import numpy as np

ROOT_SEED = 180204647

# LeNet-min shapes (BJ "conv-relu-maxpool x2, affine, softmax")
LENET_PARAM_SHAPES = (
    ("F1", (32, 1 * 5 * 5)),
    ("b1", (32,)),
    ("F2", (64, 32 * 5 * 5)),
    ("b2", (64,)),
    ("W3", (10, 64 * 7 * 7)),
    ("b3", (10,)),
)
LENET_NUM_PARAMS = sum(int(np.prod(s)) for _, s in LENET_PARAM_SHAPES)  # 83,466


# LeNet-512: SystemML's mnist_lenet.dml topology (NEXT-4; reading R22):
# ... -> affine(3136 -> 512) -> relu -> dropout -> affine(512 -> 10) -> softmax
LENET512_HIDDEN = 512
LENET512_PARAM_SHAPES = (
    ("F1", (32, 1 * 5 * 5)),
    ("b1", (32,)),
    ("F2", (64, 32 * 5 * 5)),
    ("b2", (64,)),
    ("W3", (LENET512_HIDDEN, 64 * 7 * 7)),
    ("b3", (LENET512_HIDDEN,)),
    ("W4", (10, LENET512_HIDDEN)),
    ("b4", (10,)),
)
LENET512_NUM_PARAMS = sum(int(np.prod(s)) for _, s in LENET512_PARAM_SHAPES)  # 1,663,370


def rng(*seed: int) -> np.random.Generator:
    return np.random.default_rng([ROOT_SEED, *[int(s) for s in seed]])


# ----------------------------------------------------------------------------
# family U: continuous
# ----------------------------------------------------------------------------
def uniform(shape, lo=-1.0, hi=1.0, seed=(0,)) -> np.ndarray:
    return rng(*seed).uniform(lo, hi, size=shape).astype(np.float32)


def normal(shape, std=1.0, seed=(0,)) -> np.ndarray:
    return (rng(*seed).standard_normal(size=shape) * std).astype(np.float32)


def conv_problem_U(N, C, H, W, K, R, S, P, Q, seed=(1,)):
    """X (N x CHW), F (K x CRS), b (K,), dY (N x KPQ) of family U."""
    g = rng(*seed)
    x = g.uniform(-1.0, 1.0, size=(N, C * H * W)).astype(np.float32)
    f = (g.standard_normal(size=(K, C * R * S)) * np.sqrt(2.0 / (C * R * S))).astype(np.float32)
    b = (g.standard_normal(size=(K,)) * 0.1).astype(np.float32)
    dy = g.standard_normal(size=(N, K * P * Q)).astype(np.float32)
    return x, f, b, dy


# ----------------------------------------------------------------------------
# family G: dyadic grid (exact in TF32 and in fp32 partial sums)
# ----------------------------------------------------------------------------
def dyadic(shape, lo_int, hi_int, denom, seed=(0,)) -> np.ndarray:
    """Values k/denom, k ~ U{lo_int..hi_int}; denom a power of two."""
    assert denom & (denom - 1) == 0
    k = rng(*seed).integers(lo_int, hi_int + 1, size=shape)
    return (k.astype(np.float64) / denom).astype(np.float32)


def conv_problem_G(N, C, H, W, K, R, S, P, Q, seed=(2,)):
    """Dyadic-grid conv problem: X in {-4..4}/4, F in {-3..3}/64, b in {-3..3}/16,
    dY in {-3..3}/16.  Asserts that every partial sum of fwd / bwd_filter /
    bwd_data stays below 2^22 quanta, so fp32 (and TF32-operand) accumulation is
    exact in any order."""
    x = dyadic((N, C * H * W), -4, 4, 4, seed=(*seed, 0))
    f = dyadic((K, C * R * S), -3, 3, 64, seed=(*seed, 1))
    b = dyadic((K,), -3, 3, 16, seed=(*seed, 2))
    dy = dyadic((N, K * P * Q), -3, 3, 16, seed=(*seed, 3))
    crs = C * R * S
    # quantum of products: fwd 1/(4*64); bwd_filter 1/(4*16); bwd_data 1/(64*16)
    assert crs * 1.0 * (3 / 64) * 256 + 3 / 16 * 256 < 2 ** 22
    assert N * P * Q * 1.0 * (3 / 16) * 64 < 2 ** 22
    assert K * R * S * (3 / 64) * (3 / 16) * 1024 < 2 ** 22
    return x, f, b, dy


# ----------------------------------------------------------------------------
# family M: MNIST-shaped sparse images
# ----------------------------------------------------------------------------
def mnist_like(n: int, seed=(3,)) -> np.ndarray:
    """n x 784 float32, non-zeros only in rows/cols 4..23, per-image density
    p_i ~ U(0.25, 0.50) inside the box, values k/255 with k ~ U{1..255}."""
    g = rng(*seed)
    x = np.zeros((n, 28, 28), dtype=np.float32)
    p = g.uniform(0.25, 0.50, size=(n, 1, 1))
    mask = g.random(size=(n, 20, 20)) < p
    vals = g.integers(1, 256, size=(n, 20, 20)).astype(np.float32) / np.float32(255.0)
    x[:, 4:24, 4:24] = np.where(mask, vals, np.float32(0.0))
    return x.reshape(n, 784)


def mnist_like_dyadic(n: int, seed=(4,)) -> np.ndarray:
    """MNIST-shaped support with dyadic values {1..4}/4 (family G for LeNet)."""
    g = rng(*seed)
    x = np.zeros((n, 28, 28), dtype=np.float32)
    p = g.uniform(0.25, 0.50, size=(n, 1, 1))
    mask = g.random(size=(n, 20, 20)) < p
    vals = g.integers(1, 5, size=(n, 20, 20)).astype(np.float32) / np.float32(4.0)
    x[:, 4:24, 4:24] = np.where(mask, vals, np.float32(0.0))
    return x.reshape(n, 784)


def labels(n: int, classes=10, seed=(5,)) -> np.ndarray:
    return rng(*seed).integers(0, classes, size=(n,)).astype(np.int32)


def to_csr(dense: np.ndarray):
    """Encode a dense row-major float32 matrix as CSR (row_ptr int32[rows+1],
    col_idx int32[nnz] sorted per row, val float32[nnz]); explicit zeros are
    not stored (SPEC.md matrix-core Matrix invariants).  Pure re-encoding."""
    dense = np.ascontiguousarray(dense, dtype=np.float32)
    rows, cols = dense.shape
    nz_r, nz_c = np.nonzero(dense)
    row_ptr = np.zeros(rows + 1, dtype=np.int64)
    np.add.at(row_ptr, nz_r + 1, 1)
    row_ptr = np.cumsum(row_ptr).astype(np.int32)
    return row_ptr, nz_c.astype(np.int32), dense[nz_r, nz_c].astype(np.float32)


# ----------------------------------------------------------------------------
# LeNet parameters
# ----------------------------------------------------------------------------
def lenet_params(seed=(6,), dyadic_grid=False) -> np.ndarray:
    """Flat float32[83,466] in the order F1,b1,F2,b2,W3,b3.

    Default: Glorot-uniform weights U(+-sqrt(6/(fan_in+fan_out))), zero biases
    (SPEC.md nn-layers DESIGN DECISIONS).  ``dyadic_grid``: the family-G LeNet
    grid of SURVEY.md §8(c) (F1 {-3..3}/16, F2 {-3..3}/64, W3 {-3..3}/256,
    b {-3..3}/16)."""
    g = rng(*seed)
    out = []
    for name, shape in LENET_PARAM_SHAPES:
        if dyadic_grid:
            denom = {"F1": 16, "F2": 64, "W3": 256}.get(name, 16)
            k = g.integers(-3, 4, size=shape)
            out.append((k / denom).astype(np.float32).ravel())
        elif name.startswith("b"):
            out.append(np.zeros(shape, dtype=np.float32).ravel())
        else:
            fan_out, fan_in = shape[0], shape[1]
            if name == "F1":
                fan_out = 32 * 25
            elif name == "F2":
                fan_out = 64 * 25
            lim = np.sqrt(6.0 / (fan_in + fan_out))
            out.append(g.uniform(-lim, lim, size=shape).astype(np.float32).ravel())
    flat = np.concatenate(out)
    assert flat.size == LENET_NUM_PARAMS
    return flat


def split_lenet_params(flat: np.ndarray):
    out, o = {}, 0
    for name, shape in LENET_PARAM_SHAPES:
        sz = int(np.prod(shape))
        out[name] = flat[o:o + sz].reshape(shape)
        o += sz
    return out


def lenet512_params(seed=(7,), dyadic_grid=False) -> np.ndarray:
    """Flat float32[1,663,370] in the order F1,b1,F2,b2,W3,b3,W4,b4 (LeNet-512).

    Default: Glorot-uniform weights, zero biases (as ``lenet_params``).  ``dyadic_grid``:
    F1 {-3..3}/16, F2 {-3..3}/64, W3 {-3..3}/256, W4 {-3..3}/64, b {-3..3}/16."""
    g = rng(*seed)
    out = []
    for name, shape in LENET512_PARAM_SHAPES:
        if dyadic_grid:
            denom = {"F1": 16, "F2": 64, "W3": 256, "W4": 64}.get(name, 16)
            k = g.integers(-3, 4, size=shape)
            out.append((k / denom).astype(np.float32).ravel())
        elif name.startswith("b"):
            out.append(np.zeros(shape, dtype=np.float32).ravel())
        else:
            fan_out, fan_in = shape[0], shape[1]
            if name == "F1":
                fan_out = 32 * 25
            elif name == "F2":
                fan_out = 64 * 25
            lim = np.sqrt(6.0 / (fan_in + fan_out))
            out.append(g.uniform(-lim, lim, size=shape).astype(np.float32).ravel())
    flat = np.concatenate(out)
    assert flat.size == LENET512_NUM_PARAMS
    return flat


def split_lenet512_params(flat: np.ndarray):
    out, o = {}, 0
    for name, shape in LENET512_PARAM_SHAPES:
        sz = int(np.prod(shape))
        out[name] = flat[o:o + sz].reshape(shape)
        o += sz
    return out
