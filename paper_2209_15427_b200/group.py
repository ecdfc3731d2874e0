"""Multi-GPU data parallelism over the C-ABI (qnb_group_*, include/qnb.h).

One process per GPU.  The batch is sharded in contiguous slices (rank r holds samples
[r*B, (r+1)*B)), weights are replicated, and every layer is per-sample, so the only
data-path collectives are the logits all-gather (qnb_group_forward) and the MoE expert
all-to-all (qnb_group_alltoallv).  Both are NCCL collectives issued by libqnb on the
caller's stream; the NCCL unique id is distributed by the caller (here: torch.distributed).

    group = Group.from_torch(rank, world, device)      # after dist.init_process_group
    group.forward(plan, x_shard_ptr, B, gathered_ptr, out_bytes_per_sample, stream)

`shard_bounds` / `gather_order` are the host-side bookkeeping, shared with the CPU
(gloo) tests of the data-parallel step.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L
from ._lib import check


def shard_bounds(global_batch: int, world: int, rank: int):
    """Contiguous shard of rank `rank`: [lo, hi).  The batch must split evenly (weak
    scaling keeps a fixed per-GPU batch)."""
    if global_batch % world:
        raise ValueError("global batch must be a multiple of the number of GPUs")
    b = global_batch // world
    return rank * b, (rank + 1) * b


def data_parallel_step(x_global: np.ndarray, world: int, rank: int, forward_shard, all_gather):
    """The data-parallel step bench.py runs at N > 1, backend-agnostic: this rank runs
    `forward_shard` on its slice and `all_gather(local) -> [world x local]` assembles the
    whole batch's outputs in rank order (what qnb_group_forward does with NCCL)."""
    lo, hi = shard_bounds(x_global.shape[0], world, rank)
    local = forward_shard(x_global[lo:hi])
    return np.concatenate(all_gather(local), axis=0)


class Group:
    """qnb_group: an NCCL communicator over the node's GPUs, one rank per process."""

    def __init__(self, world: int, rank: int, unique_id: bytes, device: int = 0):
        if len(unique_id) != 128:
            raise ValueError("NCCL unique id must be 128 bytes")
        self.world, self.rank = world, rank
        idb = (C.c_uint8 * 128).from_buffer_copy(unique_id)
        self.h = C.c_void_p()
        check(L.lib().qnb_group_create(world, rank, idb, device, C.byref(self.h)))

    @staticmethod
    def unique_id() -> bytes:
        idb = (C.c_uint8 * 128)()
        check(L.lib().qnb_group_unique_id(idb))
        return bytes(idb)

    @classmethod
    def from_torch(cls, rank: int, world: int, device: int) -> "Group":
        """Rank 0 draws the NCCL id; torch.distributed (any backend) broadcasts it."""
        import torch
        import torch.distributed as dist
        uid = cls.unique_id() if rank == 0 else bytes(128)
        t = torch.tensor(list(uid), dtype=torch.uint8)
        if dist.get_backend() == "nccl":
            t = t.cuda(device)
        dist.broadcast(t, 0)
        return cls(world, rank, bytes(t.cpu().tolist()), device)

    def forward(self, plan, in_ptr: int, shard_batch: int, gathered_ptr: int, out_bytes_per_sample: int,
                stream: int = 0, in_host: bool = False) -> None:
        """qnb_group_forward: this rank's shard through `plan` into its slice of `gathered`,
        then an in-place NCCL all-gather."""
        check(L.lib().qnb_group_forward(self.h, plan.h, C.c_void_p(in_ptr), shard_batch, 1 if in_host else 0,
                                        C.c_void_p(gathered_ptr), out_bytes_per_sample, C.c_void_p(stream)))

    def allgather(self, send_ptr: int, recv_ptr: int, nbytes: int, stream: int = 0) -> None:
        check(L.lib().qnb_group_allgather(self.h, C.c_void_p(send_ptr), C.c_void_p(recv_ptr), nbytes,
                                          C.c_void_p(stream)))

    def alltoallv(self, send_ptr: int, send_off, send_bytes, recv_ptr: int, recv_off, recv_bytes,
                  stream: int = 0) -> None:
        arr = lambda v: (C.c_int64 * self.world)(*[int(x) for x in v])  # noqa: E731
        check(L.lib().qnb_group_alltoallv(self.h, C.c_void_p(send_ptr), arr(send_off), arr(send_bytes),
                                          C.c_void_p(recv_ptr), arr(recv_off), arr(recv_bytes), C.c_void_p(stream)))

    def __del__(self):
        try:
            if self.h:
                L.lib().qnb_group_destroy(self.h)
        except Exception:
            pass


__all__ = ["Group", "shard_bounds", "data_parallel_step"]
