"""Data-parallel minibatch SGD plumbing (§3 "Distributed Operations": the
data-parallel plan partitions the input rows).

Host-side logic only -- every byte of compute runs in libsysml kernels:

* ``shard_rows(rank, world, global_batch)``: rank r takes the contiguous rows
  [r*B, (r+1)*B) of the global batch (the paper's row-partitioned plan).
* ``DataParallelLeNet``: one process per GPU; each rank runs
  ``sysml_lenet_step`` on its shard with ``n_global`` = the global batch, so its
  gradient buffer holds its share of the full-batch mean gradient; the library's
  in-step ``ncclAllReduce(sum)`` over torch's ProcessGroupNCCL communicator
  (NVLink/NVSwitch) makes every rank hold the full-batch gradient before the
  identical SGD update.  If the loaded NCCL cannot be resolved from inside the
  library, the same three steps run as fwd_bwd -> ``dist.all_reduce`` -> sgd.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    start: int
    stop: int

    @property
    def size(self) -> int:
        return self.stop - self.start


def shard_rows(rank: int, world: int, global_batch: int) -> Shard:
    """Contiguous, equal row shards (global_batch must divide evenly)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank/world {rank}/{world}")
    if global_batch % world:
        raise ValueError(f"global batch {global_batch} is not divisible by world size {world}")
    b = global_batch // world
    return Shard(rank, world, rank * b, (rank + 1) * b)


def allreduce_sum_(t, group=None):
    """In-place sum over the process group (host-side fallback / CPU tests)."""
    import torch.distributed as dist
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


class DataParallelLeNet:
    """One rank of the data-parallel LeNet SGD step (global batch sharded by rows)."""

    def __init__(self, global_batch: int, math: str = "tf32", group=None, net=None, sgd=None):
        """net / sgd: the per-rank LeNet handle and SGD update (default: libsysml's); the CPU
        multi-process tests pass stand-ins to exercise this host logic over gloo."""
        import torch.distributed as dist
        from . import LeNet, nccl_comm_ptr, sysml_sgd_update
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.shard = shard_rows(self.rank, self.world, global_batch)
        self.global_batch = global_batch
        self.group = group
        self.net = net if net is not None else LeNet(self.shard.size, math=math)
        self.sgd = sgd if sgd is not None else sysml_sgd_update
        self.comm: Optional[int] = None
        self.use_lib_nccl = False
        if self.world > 1 and dist.get_backend(group) == "nccl":
            import torch
            t = torch.ones(1, device="cuda")
            dist.all_reduce(t, group=group)  # creates the communicator
            self.comm = nccl_comm_ptr(group)
            self.use_lib_nccl = self.comm is not None

    def step(self, params, grads, x_local, labels_local, lr=0.01, loss_sum=None):
        from . import SysmlError
        if self.world == 1 or self.use_lib_nccl:
            try:
                self.net.step(params, grads, x_local, labels_local, self.global_batch, lr=lr,
                              nccl_comm=self.comm, loss_sum=loss_sum)
                return
            except SysmlError as e:
                if e.status != 5:  # SYSML_ERR_NCCL -> fall back to torch's all_reduce
                    raise
                self.use_lib_nccl = False
        self.net.fwd_bwd(params, x_local, labels_local, self.global_batch, grads, loss_sum)
        allreduce_sum_(grads, self.group)  # loss_sum stays this rank's share, as in the library path
        self.sgd(params, grads, lr)
