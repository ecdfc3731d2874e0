"""Expert-parallel dispatch of the MoE executor (paper_2209_15427_b200.moe.ExpertExchange)
on CPU: the host bookkeeping, and a world_size-2 gloo run whose routed result must
equal the single-process PER_SAMPLE result (src/moe.cpp:220-251) exactly."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2209_15427_b200.moe import ExpertExchange, split_moe_graph
from paper_2209_15427_b200 import graph as G, graphs

E, K, B, DIM = 4, 2, 6, 5


def route(idx):
    """qnb_moe_route restated: pairs grouped per expert, (sample, k) order inside."""
    flat = idx.reshape(-1)
    order = np.concatenate([np.nonzero(flat == e)[0] for e in range(E)]).astype(np.int64)
    counts = np.bincount(flat, minlength=E).astype(np.int64)
    slot = np.empty_like(order)
    slot[order] = np.arange(len(order))
    return counts, order // K, slot


def expert_fn(e, x):
    return x * np.float32(e + 1) + np.float32(e)


def local_result(x, idx, w):
    counts, pair_sample, slot = route(idx)
    rows = x[pair_sample]
    y = np.empty_like(rows)
    off = 0
    for e in range(E):
        y[off:off + counts[e]] = expert_fn(e, rows[off:off + counts[e]])
        off += counts[e]
    out = np.zeros((B, DIM), np.float32)
    for s in range(B):
        acc = np.zeros(DIM, np.float32)
        for k in range(K):
            acc = acc + w[s, k] * y[slot[s * K + k]]
        out[s] = acc
    return out


def rank_inputs(rank):
    rng = np.random.default_rng(100 + rank)
    x = rng.standard_normal((B, DIM)).astype(np.float32)
    idx = np.stack([rng.choice(E, K, replace=False) for _ in range(B)]).astype(np.int64)
    w = rng.uniform(0, 1, (B, K)).astype(np.float32)
    return x, idx, w


def test_plan_bookkeeping():
    counts_all = np.array([[2, 1, 0, 3], [1, 0, 2, 2]], np.int64)  # rank x expert
    send, recv, perm, local = ExpertExchange.plan(counts_all, rank=1, per_rank=2)
    assert send == [1, 4]                  # rank 1 sends e0,e1 pairs to rank 0, e2,e3 to itself
    assert recv == [3, 4]                  # rank 0 sends 0 + 3, rank 1 keeps 2 + 2
    assert local.tolist() == [2, 5]        # e2: 0 + 2, e3: 3 + 2
    # received rows: src0 [e3 e3 e3], src1 [e2 e2 e3 e3]  ->  grouped e2: src1 rows 3,4; e3: src0 0,1,2, src1 5,6
    assert perm.tolist() == [3, 4, 0, 1, 2, 5, 6]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x, idx, w = rank_inputs(rank)
        counts, pair_sample, slot = route(idx)
        xchg = ExpertExchange(E, rank, world)
        rows, local_counts = xchg.dispatch(torch.from_numpy(x[pair_sample]), counts)
        y = rows.clone()
        off = 0
        for j, e in enumerate(range(rank * xchg.per_rank, (rank + 1) * xchg.per_rank)):
            c = int(local_counts[j])
            y[off:off + c] = torch.from_numpy(expert_fn(e, rows[off:off + c].numpy()))
            off += c
        back = xchg.combine(y).numpy()
        out = np.zeros((B, DIM), np.float32)
        for s in range(B):
            acc = np.zeros(DIM, np.float32)
            for k in range(K):
                acc = acc + w[s, k] * back[slot[s * K + k]]
            out[s] = acc
        q.put((rank, np.array_equal(out, local_result(x, idx, w)), None))
    except Exception as e:  # reported to the parent
        q.put((rank, False, repr(e)))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_dispatch_matches_single_process():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, err in res:
        assert ok, f"rank {rank}: {err}"


def test_split_moe_graph_alexnet_moe():
    g = G.override_precision(graphs.alexnet_moe(1), "int8")
    trunk, moe, tail = split_moe_graph(g)
    assert G.sinks(trunk) == [moe["bottom"][0]]
    assert tail["layers"][0]["kind"] == "input" and tail["layers"][0]["top"] == moe["top"]
    assert tail["layers"][0]["top_data_type"] == "int8"
    assert G.sinks(tail) == ["prob"]
    assert G.infer_blobs(tail)["moe"]["shape"] == [1, 2048]
