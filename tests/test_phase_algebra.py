"""CPU check of the phase-split reading the product uses for strided R, S > 1 convolutions
(DESIGN.md §4 R21; paper_1802_04647_b200/csrc/phase.cu).  The identity is checked here on the
fp64 oracle, independently of the CUDA path: a strided, padded conv equals the
stride-1, pad-0 conv of the phase-split input X' with the phase-split filter F', and the two
backward operators are the corresponding gathers of the stride-1 results.  The split itself is
written out below from its definition (test code, not shared with csrc/)."""
import numpy as np
import pytest

import oracle
import synth


def split_x(x, N, C, H, W, sh, sw, ph, pw, H2, W2, C2):
    """X'[n][(a*sw + b)*C + c][h'][w'] = Xp[n][c][h'*sh + a][w'*sw + b], 0 outside Xp."""
    X = x.reshape(N, C, H, W)
    out = np.zeros((N, C2, H2, W2))
    for a in range(sh):
        for b in range(sw):
            for h2 in range(H2):
                h = h2 * sh + a - ph
                if not 0 <= h < H:
                    continue
                for w2 in range(W2):
                    w = w2 * sw + b - pw
                    if 0 <= w < W:
                        out[:, (a * sw + b) * C:(a * sw + b + 1) * C, h2, w2] = X[:, :, h, w]
    return out.reshape(N, -1)


def split_f(f, K, C, R, S, sh, sw, R2, S2, C2):
    """F'[k][(a*sw + b)*C + c][r'][s'] = F[k][c][r'*sh + a][s'*sw + b], 0 past R, S."""
    F = f.reshape(K, C, R, S)
    out = np.zeros((K, C2, R2, S2))
    for a in range(sh):
        for b in range(sw):
            for r2 in range(R2):
                for s2 in range(S2):
                    r, s = r2 * sh + a, s2 * sw + b
                    if r < R and s < S:
                        out[:, (a * sw + b) * C:(a * sw + b + 1) * C, r2, s2] = F[:, :, r, s]
    return out.reshape(K, -1)


CASES = [  # N, C, H, W, K, R, S, (sh, sw), (ph, pw)
    (2, 3, 13, 12, 4, 7, 7, (2, 2), (3, 3)),   # stem-like
    (2, 4, 9, 9, 5, 3, 3, (2, 2), (1, 1)),     # 3x3/2
    (1, 2, 10, 11, 3, 3, 3, (2, 2), (1, 1)),   # floor drops the last row / column
    (2, 2, 11, 13, 3, 5, 3, (3, 3), (2, 1)),   # stride 3, rectangular
    (1, 3, 12, 10, 2, 3, 3, (2, 1), (1, 1)),   # asymmetric stride
    (2, 3, 9, 9, 4, 2, 2, (2, 2), (0, 0)),     # R' = S' = 1 (a 1x1 over the phase channels)
]


@pytest.mark.parametrize("case", CASES)
def test_phase_split_identity(case):
    N, C, H, W, K, R, S, (sh, sw), (ph, pw) = case
    P, Q = oracle.out_extent(H, ph, R, sh), oracle.out_extent(W, pw, S, sw)
    R2, S2 = -(-R // sh), -(-S // sw)
    H2, W2 = P + R2 - 1, Q + S2 - 1
    C2 = -(-(sh * sw * C) // 8) * 8  # the product pads the phase channels to a multiple of 8
    x, f, b, dy = synth.conv_problem_U(N, C, H, W, K, R, S, P, Q, seed=(31, R, sh))
    x, f, b, dy = (t.astype(np.float64) for t in (x, f, b, dy))
    xp = split_x(x, N, C, H, W, sh, sw, ph, pw, H2, W2, C2)
    fp = split_f(f, K, C, R, S, sh, sw, R2, S2, C2)

    # forward: strided conv == stride-1, pad-0 conv over the phases
    y = oracle.conv2d_fwd(x, f, N, C, H, W, K, R, S, (sh, sw), (ph, pw), bias=b)
    y2 = oracle.conv2d_fwd(xp, fp, N, C2, H2, W2, K, R2, S2, (1, 1), (0, 0), bias=b)
    np.testing.assert_allclose(y2, y, rtol=0, atol=1e-12 * np.abs(y).max())

    # bwd_data: dX is the transpose of the split applied to dX' (a gather; rows no output
    # reads receive 0)
    dx = oracle.conv2d_bwd_data(f, dy, N, C, H, W, K, R, S, (sh, sw), (ph, pw)).reshape(N, C, H, W)
    dxp = oracle.conv2d_bwd_data(fp, dy, N, C2, H2, W2, K, R2, S2, (1, 1), (0, 0)).reshape(N, C2, H2, W2)
    got = np.zeros_like(dx)
    for h in range(H):
        for w in range(W):
            h2, a = divmod(h + ph, sh)
            w2, bb = divmod(w + pw, sw)
            if h2 < H2 and w2 < W2:
                got[:, :, h, w] = dxp[:, (a * sw + bb) * C:(a * sw + bb + 1) * C, h2, w2]
    np.testing.assert_allclose(got, dx, rtol=0, atol=1e-12 * np.abs(dx).max())

    # bwd_filter: dF[k,c,r,s] = dF'[k][(r%sh, s%sw, c)][r/sh][s/sw]; db unchanged
    df, db = oracle.conv2d_bwd_filter(x, dy, N, C, H, W, K, R, S, (sh, sw), (ph, pw))
    dfp, dbp = oracle.conv2d_bwd_filter(xp, dy, N, C2, H2, W2, K, R2, S2, (1, 1), (0, 0))
    dfp = dfp.reshape(K, C2, R2, S2)
    got = np.zeros((K, C, R, S))
    for r in range(R):
        for s in range(S):
            c0 = ((r % sh) * sw + s % sw) * C
            got[:, :, r, s] = dfp[:, c0:c0 + C, r // sh, s // sw]
    np.testing.assert_allclose(got.reshape(K, -1), df, rtol=0, atol=1e-12 * np.abs(df).max())
    np.testing.assert_allclose(dbp, db, rtol=0, atol=1e-12 * np.abs(db).max())
