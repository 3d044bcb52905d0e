"""CPU (gloo, world_size 2) tests of the data-parallel host logic.

The per-rank compute here is the fp64 oracle (test infrastructure); what is under test
is the plumbing the GPU path uses: contiguous row shards, gradients pre-scaled by
1/n_global, the sum-allreduce over the process group, and the identical SGD update
-- i.e. that the sharded step reproduces the full-batch step."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_1802_04647_b200.dp import allreduce_sum_, shard_rows


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_rows():
    assert [shard_rows(r, 4, 8192).start for r in range(4)] == [0, 2048, 4096, 6144]
    assert shard_rows(3, 4, 8192).stop == 8192
    assert shard_rows(0, 1, 64).size == 64
    with pytest.raises(ValueError):
        shard_rows(0, 3, 64)
    with pytest.raises(ValueError):
        shard_rows(2, 2, 64)


def _worker(rank, world, port, gb, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x = synth.mnist_like(gb, seed=(50,))
        y = synth.labels(gb, seed=(51,))
        prm = synth.lenet_params(seed=(52,)).astype(np.float64)
        sh = shard_rows(rank, world, gb)
        g, loss = oracle.lenet_fwd_bwd(x[sh.start:sh.stop], y[sh.start:sh.stop], prm, n_global=gb)
        gt = torch.from_numpy(g.copy())
        lt = torch.tensor([loss], dtype=torch.float64)
        allreduce_sum_(gt)
        allreduce_sum_(lt)
        new = oracle.sgd_update(prm, gt.numpy(), 0.01)
        out_q.put((rank, new, lt.item()))
    finally:
        dist.destroy_process_group()


def test_two_rank_sharded_step_equals_full_batch():
    gb, world = 6, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, gb, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda t: t[0])
    # every rank ends with bitwise-identical parameters (identical update on the reduced grads)
    assert np.array_equal(res[0][1], res[1][1])
    x = synth.mnist_like(gb, seed=(50,))
    y = synth.labels(gb, seed=(51,))
    prm = synth.lenet_params(seed=(52,)).astype(np.float64)
    g, loss = oracle.lenet_fwd_bwd(x, y, prm, n_global=gb)
    np.testing.assert_allclose(res[0][1], oracle.sgd_update(prm, g, 0.01), rtol=0, atol=1e-15)
    assert abs(res[0][2] - loss) <= 1e-14


class _OracleNet:
    """CPU stand-in for the per-rank libsysml LeNet handle: the fp64 oracle's fwd_bwd on the
    rank's rows (so DataParallelLeNet's own step logic runs over gloo without a GPU)."""

    def __init__(self):
        self.calls = []

    def fwd_bwd(self, params, x, labels, n_global, grads, loss_sum=None):
        self.calls.append((x.shape[0], n_global))
        g, loss = oracle.lenet_fwd_bwd(x.numpy(), labels.numpy(), params.numpy(), n_global=n_global)
        grads.copy_(torch.from_numpy(g))
        if loss_sum is not None:
            loss_sum.fill_(loss)


def _dp_worker(rank, world, port, gb, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1802_04647_b200.dp import DataParallelLeNet
        net = _OracleNet()
        dp = DataParallelLeNet(gb, net=net, sgd=lambda p, g, lr: p.sub_(lr * g))
        assert (dp.world, dp.rank, dp.use_lib_nccl) == (world, rank, False)
        x = synth.mnist_like(gb, seed=(53,))
        y = synth.labels(gb, seed=(54,))
        prm = torch.from_numpy(synth.lenet_params(seed=(55,)).astype(np.float64))
        grads = torch.zeros_like(prm)
        for it in range(2):  # two steps: the second starts from the reduced, updated parameters
            sh = dp.shard
            dp.step(prm, grads, torch.from_numpy(x[sh.start:sh.stop]), torch.from_numpy(y[sh.start:sh.stop]),
                    lr=0.01)
        out_q.put((rank, prm.numpy().copy(), net.calls))
    finally:
        dist.destroy_process_group()


def test_data_parallel_lenet_step_logic_over_gloo():
    """DataParallelLeNet.step itself (not a re-implementation) at world size 2 over gloo:
    each rank computes its contiguous shard with n_global = the global batch, the gradients
    are sum-allreduced, the identical update runs on every rank; two steps match two
    full-batch oracle steps and both ranks hold bitwise-identical parameters."""
    gb, world = 8, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dp_worker, args=(r, world, port, gb, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda t: t[0])
    assert np.array_equal(res[0][1], res[1][1])
    assert res[0][2] == [(4, 8), (4, 8)] and res[1][2] == [(4, 8), (4, 8)]
    x = synth.mnist_like(gb, seed=(53,))
    y = synth.labels(gb, seed=(54,))
    prm = synth.lenet_params(seed=(55,)).astype(np.float64)
    for _ in range(2):
        g, _l = oracle.lenet_fwd_bwd(x, y, prm, n_global=gb)
        prm = oracle.sgd_update(prm, g, 0.01)
    np.testing.assert_allclose(res[0][1], prm, rtol=0, atol=1e-14)
