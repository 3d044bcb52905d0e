"""Time the LeNet step replayed from a CUDA graph at a given local batch.
usage: time_step_graph.py [batch]"""
import sys, os, statistics
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
cs = torch.cuda.Stream()
cs.wait_stream(torch.cuda.current_stream())
gr = torch.cuda.CUDAGraph()
with torch.cuda.graph(gr, stream=cs):
    net.step(prm, g, x, y, 8192)
torch.cuda.current_stream().wait_stream(cs)
for _ in range(3):
    gr.replay()
torch.cuda.synchronize()
ts = []
for _ in range(20):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); gr.replay(); b.record(); b.synchronize()
    ts.append(a.elapsed_time(b))
ms = statistics.median(ts)
print(f"graph batch {n}: {ms*1e3:.1f} us/step  {n/ms*1e3/1e6:.2f} M img/s per GPU")
