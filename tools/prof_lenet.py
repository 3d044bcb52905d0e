"""ncu target: a few LeNet fwd_bwd steps.  usage: prof_lenet.py [batch] [math] [csr]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_1802_04647_b200 as S
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
math = sys.argv[2] if len(sys.argv) > 2 else "tf32"
csr = len(sys.argv) > 3 and sys.argv[3] == "csr"
x = synth.mnist_like(n, seed=(3,))
y = torch.from_numpy(synth.labels(n, seed=(4,))).cuda()
prm = torch.from_numpy(synth.lenet_params(seed=(5,))).cuda()
g = torch.empty_like(prm)
net = S.LeNet(n, math=math, csr=csr, max_nnz=n * 784)
if csr:
    xs = torch.from_numpy(x).cuda().to_sparse_csr()
    xin = S.CSR(xs.crow_indices().int(), xs.col_indices().int(), xs.values().float(), n, 784)
else:
    xin = torch.from_numpy(x).cuda()
for _ in range(3):
    net.fwd_bwd(prm, xin, y, n, g)
torch.cuda.synchronize()
print("ok")
