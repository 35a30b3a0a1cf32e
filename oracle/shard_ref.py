"""CPU shard double for the multi-GPU protocol — TEST INFRASTRUCTURE ONLY.

Implements the shard contract of paper_2507_14222_b200/sharded.py (enumerate →
all-to-all → receive → finish → partial_evidence) on the host with numpy and
the plain-C oracle, following the same protocol as the device shard
(include/ig_b200.h "multi-GPU"): distinct canonical rows, 64x64 tiles of the
u <= v triangle dealt round-robin to ranks, local exact dedup, owner = content
hash mod world, owner-side exact dedup, support / coverage against the full
replicated class rows.  Lets tests/test_sharded_cpu.py drive the product's
torch.distributed orchestration under gloo on CPU.
"""
from __future__ import annotations

import hashlib

import numpy as np

from oracle import oracle

TILE = 64


def canonical_distinct(rows: np.ndarray) -> np.ndarray:
    if rows.shape[0] == 0:
        return rows
    u = np.unique(rows.view(np.uint64), axis=0)
    order = np.lexsort(u.T[::-1])
    return u[order].view(np.int64)


def tile_of(t: int):
    j = int((np.sqrt(8.0 * t + 1.0) - 1.0) / 2.0)
    while j * (j + 1) // 2 > t:
        j -= 1
    while (j + 1) * (j + 2) // 2 <= t:
        j += 1
    return t - j * (j + 1) // 2, j


def owner_of(content: bytes, world: int) -> int:
    return int.from_bytes(hashlib.blake2b(content, digest_size=8).digest(), "little") % world


class RefShard:
    def __init__(self, ctx, enc, rank: int, world: int, config=None):
        # enc: dict(attack=..., normal=...) numpy rows (replicated on every rank)
        self.rank, self.world = rank, world
        self.X = [np.ascontiguousarray(enc["attack"]), np.ascontiguousarray(enc["normal"])]
        self.U = [canonical_distinct(x) for x in self.X]
        self.owned = [None, None]
        self.pure = [None, None]

    def enumerate(self, cls: int):
        import torch
        U = self.U[cls]
        m = U.shape[0]
        blocks = (m + TILE - 1) // TILE
        n_tiles = blocks * (blocks + 1) // 2
        local = {}
        for t in range(self.rank, n_tiles, self.world):
            bi, bj = tile_of(t)
            for u in range(bi * TILE, min(m, bi * TILE + TILE)):
                for v in range(max(u, bj * TILE), min(m, bj * TILE + TILE)):
                    c = U[u] & U[v]
                    if not c.any():
                        continue
                    local.setdefault(c.tobytes(), (u, v))
        buckets = [[] for _ in range(self.world)]
        for content, (u, v) in local.items():
            buckets[owner_of(content, self.world)].append(u | (v << 32))
        counts = [len(b) for b in buckets]
        send = torch.tensor([x for b in buckets for x in b], dtype=torch.int64)
        return counts, send

    def receive(self, cls: int, recv, n_records: int) -> None:
        U = self.U[cls]
        seen = {}
        for x in recv[:n_records].tolist():
            u, v = x & 0xffffffff, x >> 32
            c = U[u] & U[v]
            seen.setdefault(c.tobytes(), c)
        k = U.shape[1]
        rows = np.stack(list(seen.values())) if seen else np.zeros((0, k), np.int64)
        self.owned[cls] = canonical_distinct(rows) if len(rows) else rows

    def finish(self):
        totals = []
        for c in range(2):
            w = self.owned[c]
            sup = oracle.count_support(w, self.X[c]) if len(w) else np.zeros(0, np.int64)
            sc = oracle.score_patterns(w, sup) if len(w) else np.zeros(0, np.int64)
            keep = oracle.coverage_any(w, self.X[1 - c]) == 0 if len(w) else np.zeros(0, bool)
            self.pure[c] = oracle.Dictionary(w[keep], sup[keep], sc[keep])
            totals.append(int(sc.sum()))
        return tuple(totals)

    @property
    def model(self):
        return self.pure

    def partial_evidence(self, tests: np.ndarray):
        import torch
        out = []
        for c in range(2):
            d = self.pure[c]
            v = oracle.fused_score(d.words, d.scores, tests) if len(d.words) else np.zeros(len(tests), np.int64)
            out.append(torch.tensor(v, dtype=torch.int64))
        return out[0], out[1]
