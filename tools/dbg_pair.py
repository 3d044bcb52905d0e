"""Route check for the pair conv kernel on the forced-test shapes (debug helper)."""
import numpy as np, torch, synth, paper_1802_04647_b200 as S
from tests.test_gpu_parity import dev, host
shapes = [(3, 64, 14, 14, 256, 3, 1), (2, 32, 9, 11, 512, 3, 1), (3, 128, 7, 7, 256, 1, 0),
          (2, 256, 14, 14, 64, 3, 1), (2, 256, 8, 8, 128, 1, 0), (1, 16, 5, 6, 256, 3, 1)]
for i, (N, C, H, W, K, R, pd) in enumerate(shapes):
    P, Q = H + 2 * pd - R + 1, W + 2 * pd - R + 1
    x, f, b, dy = synth.conv_problem_U(N, C, H, W, K, R, R, P, Q, seed=(990 + i,))
    d = S.conv_desc(N, C, H, W, K, R, R, 1, pd, "tf32")
    S.sysml_conv2d(dev(x), dev(f), d, bias=dev(b)); print(i, "fwd", S.sysml_last_route())
    S.sysml_conv2d_bwd_data(dev(f), dev(dy), d); print(i, "bwd", S.sysml_last_route())
