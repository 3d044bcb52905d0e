"""Per-stage device times of the LeNet step at a given local batch.  usage: stage_times.py [batch]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_1802_04647_b200 as S
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
x = torch.from_numpy(synth.mnist_like(n, seed=(3,))).cuda()
y = torch.from_numpy(synth.labels(n, seed=(4,))).cuda()
prm = torch.from_numpy(synth.lenet_params(seed=(5,))).cuda()
g = torch.empty_like(prm)
net = S.LeNet(n, math="tf32")
for _ in range(3):
    net.step(prm, g, x, y, 8192)
torch.cuda.synchronize()
net.set_timing(True); net.get_timing(reset=True)
for _ in range(10):
    net.step(prm, g, x, y, 8192)
torch.cuda.synchronize()
t = net.get_timing()
tot = 0.0
for k, (ms, c) in t.items():
    if c:
        print(f"{k:34s} {ms / c * 1e3:8.1f} us")
        tot += ms / c
print(f"{'sum':34s} {tot * 1e3:8.1f} us")
