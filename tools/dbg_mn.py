import sys, os
sys.path.insert(0, "/root/repo")
import numpy as np, torch, synth
import paper_1802_04647_b200 as S
N, C, H, W, K = 2, 16, 4, 8, 16
x = np.zeros((N, C * H * W), np.float32)
f = np.zeros((K, C), np.float32)
# x[n,c,pos] = pos + 100*c ; f = identity -> y[n,k,pos] = x[n,k,pos]
for n in range(N):
    for c in range(C):
        x[n, c*H*W:(c+1)*H*W] = np.arange(H*W) + 100*c + 1000*n
for k in range(K): f[k, k] = 1.0
d = S.conv_desc(N, C, H, W, K, 1, 1, 1, 0, "tf32")
y = S.sysml_conv2d(torch.from_numpy(x).cuda(), torch.from_numpy(f).cuda(), d).cpu().numpy()
print("max err", np.abs(y - x).max())
yy = y.reshape(N, K, H*W)
np.set_printoptions(linewidth=200)
print(yy[0, :3, :12])
print(yy[0, 8:10, :12])
