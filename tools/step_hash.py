"""Run K LeNet steps (eager, then graph-replayed) and print a hash of the final parameters
and loss -- the step is deterministic, so any launch-ordering change (e.g. SYSML_PDL=0/1)
must give identical hashes.  usage: step_hash.py [batch] [steps] [csr]"""
import sys, os, hashlib
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_1802_04647_b200 as S
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
K = int(sys.argv[2]) if len(sys.argv) > 2 else 10
csr = len(sys.argv) > 3 and sys.argv[3] == "csr"
xd = synth.mnist_like(n, seed=(3,))
y = torch.from_numpy(synth.labels(n, seed=(4,))).cuda()
prm = torch.from_numpy(synth.lenet_params(seed=(5,))).cuda()
g = torch.empty_like(prm)
if csr:
    xt = torch.from_numpy(xd)
    nz = xt.nonzero()
    rp = torch.zeros(n + 1, dtype=torch.int32)
    rp[1:] = torch.cumsum(torch.bincount(nz[:, 0], minlength=n), 0).to(torch.int32)
    x = S.CSR(rp.cuda(), nz[:, 1].to(torch.int32).cuda(), xt[nz[:, 0], nz[:, 1]].contiguous().cuda(), n, 784)
    net = S.LeNet(n, math="tf32", csr=True, max_nnz=x.nnz)
else:
    x = torch.from_numpy(xd).cuda()
    net = S.LeNet(n, math="tf32")
loss = torch.zeros(1, device="cuda")
for _ in range(K):
    net.step(prm, g, x, y, 8192, loss_sum=loss)
torch.cuda.synchronize()
h1 = hashlib.sha1(prm.cpu().numpy().tobytes() + loss.cpu().numpy().tobytes()).hexdigest()[:16]
cs = torch.cuda.Stream()
cs.wait_stream(torch.cuda.current_stream())
gr = torch.cuda.CUDAGraph()
with torch.cuda.graph(gr, stream=cs):
    net.step(prm, g, x, y, 8192, loss_sum=loss)
torch.cuda.current_stream().wait_stream(cs)
for _ in range(K):
    gr.replay()
torch.cuda.synchronize()
h2 = hashlib.sha1(prm.cpu().numpy().tobytes() + loss.cpu().numpy().tobytes()).hexdigest()[:16]
print(f"batch {n} csr={csr} eager {h1} graph {h2} loss {loss.item():.6f}")
