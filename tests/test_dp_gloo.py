"""The N > 1 paths on CPU with world_size 2 over gloo: the data-parallel
step bench.py runs (contiguous batch shards + all-gather of the logits, what
qnb_group_forward does with NCCL) and MoeNet's expert-parallel step
(ExpertExchange.run: dispatch -> local experts -> combine), each with the device compute
mocked on the host, must give exactly the single-process result."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2209_15427_b200.group import data_parallel_step, shard_bounds
from paper_2209_15427_b200.moe import ExpertExchange

E, K, DIM = 4, 2, 6


def forward_mock(x):
    """A per-sample 'network': fixed linear map + softmax per row (rows independent)."""
    w = np.linspace(-1, 1, x.shape[1] * 10, dtype=np.float32).reshape(x.shape[1], 10)
    z = x @ w
    z = np.exp(z - z.max(axis=1, keepdims=True))
    return (z / z.sum(axis=1, keepdims=True)).astype(np.float32)


def expert_mock(e, rows):
    return rows * (e + 1) + e


def moe_single(x, idx, w):
    """Single-process PER_SAMPLE MoE (src/moe.cpp:220-251) with the mocked experts."""
    B = x.shape[0]
    out = np.zeros_like(x)
    for s in range(B):
        acc = np.zeros(x.shape[1], np.float32)
        for k in range(K):
            acc = acc + w[s, k] * expert_mock(int(idx[s, k]), x[s])
        out[s] = acc
    return out


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(5)
        xg = rng.standard_normal((8, DIM)).astype(np.float32)  # the global batch (same on every rank)

        def all_gather(local):
            t = torch.from_numpy(local)
            parts = [torch.empty_like(t) for _ in range(world)]
            dist.all_gather(parts, t)
            return [p.numpy() for p in parts]

        dp = data_parallel_step(xg, world, rank, forward_mock, all_gather)
        ok_dp = np.array_equal(dp, forward_mock(xg))

        # expert parallel: this rank's samples, routed pairs grouped by global expert
        lo, hi = shard_bounds(xg.shape[0], world, rank)
        x = xg[lo:hi]
        idx = np.stack([np.random.default_rng(50 + lo + s).choice(E, K, replace=False) for s in range(hi - lo)])
        wts = np.random.default_rng(90 + rank).uniform(0, 1, (hi - lo, K)).astype(np.float32)
        flat = idx.reshape(-1)
        order = np.concatenate([np.nonzero(flat == e)[0] for e in range(E)]).astype(np.int64)
        counts = np.bincount(flat, minlength=E).astype(np.int64)
        slot = np.empty_like(order)
        slot[order] = np.arange(len(order))
        xchg = ExpertExchange(E, rank, world)
        back = xchg.run(torch.from_numpy(x[order // K]), counts,
                        lambda e, r: torch.from_numpy(expert_mock(e, r.numpy()))).numpy()
        out = np.zeros_like(x)
        for s in range(x.shape[0]):
            acc = np.zeros(DIM, np.float32)
            for k in range(K):
                acc = acc + wts[s, k] * back[slot[s * K + k]]
            out[s] = acc
        ok_moe = np.array_equal(out, moe_single(x, idx, wts))
        q.put((rank, ok_dp, ok_moe, None))
    except Exception as e:  # reported to the parent
        q.put((rank, False, False, repr(e)))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_data_parallel_and_expert_parallel_steps():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, ok_dp, ok_moe, err in res:
        assert err is None, f"rank {rank}: {err}"
        assert ok_dp, f"rank {rank}: data-parallel step differs from the single-process result"
        assert ok_moe, f"rank {rank}: expert-parallel step differs from the single-process result"


def test_shard_bounds():
    assert [shard_bounds(1024, 4, r) for r in range(4)] == [(0, 256), (256, 512), (512, 768), (768, 1024)]
    with pytest.raises(ValueError):
        shard_bounds(10, 4, 0)
