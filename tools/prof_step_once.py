"""One eager LeNet step at a given local batch (for SYSML_TC_PROFILE=1 per-warp clock breakdowns)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_1802_04647_b200 as S
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
x = torch.from_numpy(synth.mnist_like(n, seed=(3,))).cuda()
y = torch.from_numpy(synth.labels(n, seed=(4,))).cuda()
prm = torch.from_numpy(synth.lenet_params(seed=(5,))).cuda()
g = torch.empty_like(prm)
net = S.LeNet(n, math="tf32")
for _ in range(2):
    net.step(prm, g, x, y, 8192)
torch.cuda.synchronize()
