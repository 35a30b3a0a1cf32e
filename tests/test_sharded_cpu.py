"""World-size-2 gloo test of the multi-GPU orchestration on CPU.

paper_2507_14222_b200/sharded.py's fit_distributed / evidence_distributed /
TorchExchange run unchanged under torch.distributed(gloo); the device shard is
replaced by the oracle-backed double (oracle/shard_ref.py) implementing the same
protocol.  The union of the ranks' owned pure dictionaries and the all-reduced
evidence must equal the single-process oracle fit exactly."""
import os
import socket

import numpy as np
import torch.multiprocessing as mp

from tests.helpers import random_rows


def _data():
    rng = np.random.default_rng(8)
    L = 150
    Xa = random_rows(rng, 170, L, 0.85)
    Xn = random_rows(rng, 150, L, 0.85)
    Xa[40:60] = Xa[0:20]  # duplicate rows
    T = random_rows(rng, 90, L, 0.9)
    return L, Xa, Xn, T


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    from oracle.shard_ref import RefShard
    from paper_2507_14222_b200 import sharded

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    L, Xa, Xn, T = _data()
    ex = sharded.TorchExchange(device=torch.device("cpu"))
    res = sharded.fit_distributed(None, {"attack": Xa, "normal": Xn}, rank, world, ex, shard_factory=RefShard)
    A, N = sharded.evidence_distributed(res, T, ex)
    pure = [(d.words.tolist(), d.supports.tolist(), d.scores.tolist()) for d in res.shard.pure]
    gathered = [None] * world
    dist.all_gather_object(gathered, pure)
    if rank == 0:
        out.put((gathered, A.tolist(), N.tolist()))
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_rank_gloo_fit_equals_oracle():
    from oracle import oracle
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    gathered, A, N = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    L, Xa, Xn, T = _data()
    ref = oracle.fit(Xa, Xn)
    for c in range(2):
        rows = [np.array(g[c][0], np.int64).reshape(-1, Xa.shape[1]) for g in gathered]
        sup = np.concatenate([np.array(g[c][1], np.int64) for g in gathered])
        sc = np.concatenate([np.array(g[c][2], np.int64) for g in gathered])
        allw = np.concatenate(rows)
        order = np.lexsort(allw.view(np.uint64).T[::-1])
        assert np.array_equal(allw[order], ref.pure[c].words)
        assert np.array_equal(sup[order], ref.pure[c].supports)
        assert np.array_equal(sc[order], ref.pure[c].scores)
        # every owned set is disjoint from the others (exact global dedup)
        assert sum(len(r) for r in rows) == len(ref.pure[c].words)
    assert A == oracle.fused_score(ref.pure[0].words, ref.pure[0].scores, T).tolist()
    assert N == oracle.fused_score(ref.pure[1].words, ref.pure[1].scores, T).tolist()
