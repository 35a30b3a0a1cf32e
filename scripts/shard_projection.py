"""Per-rank cost of the sharded fit with `world` ranks
emulated one after another on ONE B200, and the N-GPU step time it implies.

Each rank's phases run alone on the device (create = its distinct rows and
tile share; enumerate = its pair tiles + owner bucketing; receive = dedup of
the records it owns; finish = support / score / purify / order of its owned
candidates; evidence = its partial A/N), timed with a device synchronize on
both sides.  The projection for N GPUs is

    encode (replicated) + max over ranks of (create + enumerate + receive +
    finish + evidence) + all-to-all (max bytes a rank sends or receives at
    `--link-gbs`) + the A/N all-reduce (2 x n_test x 8 B ring)

This is a model, not a measurement: only one GPU is available to this build,
and the driver's own 2/4/8-GPU bench lines are the numbers that count.

    python scripts/shard_projection.py [--rows 148517] [--ratio 8] [--worlds 1,2,4,8]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2507_14222_b200 import api, sharded, synth  # noqa: E402


def _t(fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    return out, time.perf_counter() - t0


def run_world(ctx, enc, tenc, world):
    shards, create = [], []
    for r in range(world):
        sh, dt = _t(lambda: sharded.Shard(ctx, enc, r, world))
        shards.append(sh)
        create.append(dt)
    enum = [[0.0, 0.0] for _ in range(world)]
    recv_t = [[0.0, 0.0] for _ in range(world)]
    sent = [0] * world
    got = [0] * world
    for cls in range(2):
        outs = []
        for r, sh in enumerate(shards):
            (counts, send), dt = _t(lambda: sh.enumerate(cls))
            enum[r][cls] = dt
            outs.append((counts, send.clone()))
            sent[r] += 8 * (sum(counts) - counts[r])
        for r, sh in enumerate(shards):
            parts = [t[sum(c[:r]):sum(c[:r]) + c[r]] for c, t in outs]
            recv = torch.cat(parts)
            got[r] += 8 * sum(c[r] for i, (c, _) in enumerate(outs) if i != r)
            _, dt = _t(lambda: sh.receive(cls, recv, int(recv.numel())))
            recv_t[r][cls] = dt
        del outs
    finish, evid = [], []
    for sh in shards:
        _, dt = _t(sh.finish)
        finish.append(dt)
        _, dt = _t(lambda: sh.partial_evidence(tenc))
        evid.append(dt)
    per_rank = [create[r] + sum(enum[r]) + sum(recv_t[r]) + finish[r] + evid[r] for r in range(world)]
    del shards
    return dict(create=create, enumerate=enum, receive=recv_t, finish=finish, evidence=evid, per_rank=per_rank,
                sent_bytes=sent, recv_bytes=got)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=148517)
    ap.add_argument("--ratio", type=int, default=8)
    ap.add_argument("--worlds", default="1,2,4,8")
    ap.add_argument("--link-gbs", type=float, default=400.0, help="effective all-to-all GB/s per GPU (assumed)")
    args = ap.parse_args()
    csv = synth.nsl_csv(args.rows, seed=2507)
    ctx = api.default_context()
    table = api.read_csv(csv)
    ntr = args.ratio * table.rows // 10
    tr, te = table.slice(0, ntr), table.slice(ntr, table.rows)
    schema = api.infer_schema(tr, "label", decimals=1)
    ctr, cte = api.Columns(tr, schema, True).upload(ctx), api.Columns(te, schema, False).upload(ctx)
    for _ in range(4):  # the first encodes of a process grow the memory pool
        enc, t_enc = _t(lambda: api.encode_training(ctr, ctx))
        tenc, t_tenc = _t(lambda: api.encode_rows(cte, enc, ctx))
    # single-device reference step: the fused fit + evidence
    for _ in range(3):
        res, t_single = _t(lambda: api.fit_evidence_encoded(enc, tenc))
        del res  # a live C4 model makes the shards' allocations grow the pool
    n_test = tenc.rows(2)
    for world in [int(w) for w in args.worlds.split(",")]:
        run_world(ctx, enc, tenc, world)  # warm the pool for this world size
        w = run_world(ctx, enc, tenc, world)
        xfer = max(max(w["sent_bytes"]), max(w["recv_bytes"])) / (args.link_gbs * 1e9)
        allreduce = 2 * 2 * n_test * 8 * (world - 1) / world / (args.link_gbs * 1e9) if world > 1 else 0.0
        proj = t_enc + t_tenc + max(w["per_rank"]) + xfer + allreduce
        print(json.dumps({
            "rows": args.rows, "ratio": f"{args.ratio}|{10 - args.ratio}", "world": world,
            "single_device_fit_evidence_ms": round(1e3 * t_single, 2),
            "encode_ms": round(1e3 * (t_enc + t_tenc), 2),
            "max_rank_ms": round(1e3 * max(w["per_rank"]), 2),
            "min_rank_ms": round(1e3 * min(w["per_rank"]), 2),
            "phases_max_ms": {k: round(1e3 * max(sum(x) if isinstance(x, list) else x for x in w[k]), 2)
                              for k in ("create", "enumerate", "receive", "finish", "evidence")},
            "all_to_all_max_mb": round(max(max(w["sent_bytes"]), max(w["recv_bytes"])) / 1e6, 1),
            "projected_step_ms": round(1e3 * proj, 2),
            "projected_speedup_vs_1gpu": round((t_enc + t_tenc + t_single) / proj, 2),
            "link_gbs_assumed": args.link_gbs,
        }), flush=True)


if __name__ == "__main__":
    main()
