"""Debug helper: tcgen05 bwd_filter vs oracle on small shapes (prints error stats)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, synth
import paper_1802_04647_b200 as S

cases = [
    # N, C, H, W, K, R, S, pad
    (1, 16, 8, 8, 128, 1, 1, 0),
    (1, 16, 8, 8, 64, 1, 1, 0),
    (1, 16, 8, 8, 128, 3, 3, 1),
    (2, 32, 14, 14, 64, 5, 5, 2),
    (1, 16, 8, 8, 64, 2, 1, 0),
    (1, 32, 6, 6, 64, 1, 1, 0),
]
for (N, C, H, W, K, R, S_, pd) in cases:
    P = H + 2 * pd - R + 1; Q = W + 2 * pd - S_ + 1
    x, f, b, dy = synth.conv_problem_G(N, C, H, W, K, R, S_, P, Q)
    d = S.conv_desc(N, C, H, W, K, R, S_, 1, pd, "tf32")
    df, db = S.sysml_conv2d_bwd_filter(torch.from_numpy(x).cuda(), torch.from_numpy(dy).cuda(), d)
    dfr, dbr = oracle.conv2d_bwd_filter(x, dy, N, C, H, W, K, R, S_, (1, 1), (pd, pd))
    g = df.cpu().numpy().astype(np.float64)
    err = np.abs(g - dfr)
    bad = np.argwhere(err > 1e-6)
    print((N, C, H, W, K, R, S_, pd), "max err", err.max(), "max ref", np.abs(dfr).max(),
          "nbad", len(bad), "of", err.size, "db err", np.abs(db.cpu().numpy() - dbr).max())
    if len(bad):
        dfr4 = dfr.reshape(K, C, R, S_); g4 = g.reshape(K, C, R, S_)
        bad4 = np.argwhere(np.abs(g4 - dfr4) > 1e-6)
        print("   first bad (k,c,r,s):", bad4[:6].tolist())
        print("   gpu/ref at first bad:", [(g4[tuple(i)], dfr4[tuple(i)]) for i in bad4[:4]])
        # is the gpu result another (r,s) / k permutation of the ref?
        print("   zero fraction gpu:", np.mean(g == 0), "ref:", np.mean(dfr == 0))
