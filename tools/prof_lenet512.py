"""Eager LeNet-512 steps at a given local batch (for ncu launch lists / captures)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_1802_04647_b200 as S
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
x = torch.from_numpy(synth.mnist_like(n, seed=(3,))).cuda()
y = torch.from_numpy(synth.labels(n, seed=(4,))).cuda()
prm = torch.from_numpy(synth.lenet512_params(seed=(5,))).cuda()
g = torch.empty_like(prm)
net = S.LeNet(n, math="tf32", model="lenet512", keep_p=0.5, seed=1)
for _ in range(steps):
    net.step(prm, g, x, y, n)
torch.cuda.synchronize()
