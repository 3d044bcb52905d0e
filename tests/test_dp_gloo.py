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
