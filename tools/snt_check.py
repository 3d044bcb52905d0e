"""SN-mode conv parity under the SYSML_TC_SNT setting of the environment (read once per
process): bwd_data / fwd shapes whose output has <= 32 channels, TF32, vs the fp64 oracle."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, oracle, synth
import paper_1802_04647_b200 as S
worst = 0.0
for (N, C, H, W, K, R, pd) in [(3, 64, 14, 14, 32, 5, 2), (2, 48, 9, 11, 16, 5, 2), (2, 40, 12, 10, 32, 3, 1),
                               (5, 32, 14, 14, 32, 5, 2), (64, 64, 14, 14, 32, 5, 2)]:
    P, Q = H + 2 * pd - R + 1, W + 2 * pd - R + 1
    x, f, b, dy = synth.conv_problem_U(N, C, H, W, K, R, R, P, Q, seed=(77,))
    d = S.conv_desc(N, C, H, W, K, R, R, 1, pd, "tf32")
    y = S.sysml_conv2d(torch.from_numpy(x).cuda(), torch.from_numpy(f).cuda(), d, bias=torch.from_numpy(b).cuda())
    r1 = S.sysml_last_route()
    ref = oracle.conv2d_fwd(x, f, N, C, H, W, K, R, R, (1, 1), (pd, pd), bias=b)
    e1 = np.abs(y.cpu().numpy() - ref).max() / np.abs(ref).max()
    # bwd_data with C and K swapped so the OUTPUT has K channels (SN applies to <= 32 outputs)
    d2 = S.conv_desc(N, K, H, W, C, R, R, 1, pd, "tf32")
    f2 = synth.normal((C, K * R * R), 0.1, seed=(78,))
    dy2 = synth.normal((N, C * P * Q), seed=(79,))
    dx = S.sysml_conv2d_bwd_data(torch.from_numpy(f2).cuda(), torch.from_numpy(dy2).cuda(), d2)
    r2 = S.sysml_last_route()
    ref2 = oracle.conv2d_bwd_data(f2, dy2, N, K, H, W, C, R, R, (1, 1), (pd, pd))
    e2 = np.abs(dx.cpu().numpy() - ref2).max() / np.abs(ref2).max()
    torch.cuda.synchronize()
    print(f"{(N, C, H, W, K, R)} fwd {e1:.2e} [{r1}]  bwd_data {e2:.2e} [{r2}]")
    worst = max(worst, e1, e2)
print("SNT", os.environ.get("SYSML_TC_SNT"), "worst", worst, "OK" if worst <= 5e-3 else "FAIL")
