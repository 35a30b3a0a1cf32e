#!/usr/bin/env python
"""IG fit benchmark on synthetic NSL-KDD-shape data (BASELINE.json `metric`).

Workload (BASELINE.json configs[2], the paper's Table 2 setting):
148,517 synthetic NSL-KDD-shape records, 41 columns + label, p = 1 decimal,
positional 10/90 train/test split (14,851 train / 133,666 test).

One step = the whole IG train-and-evaluate hot path on that batch:
  kernel (1) tokenise + vocabulary + anti-contradiction + pack (train and test rows),
  kernels (2)-(5) enumerate → dedup → support/score → canonical order → purify,
  kernel (6) evidence A/N for all 133,666 test rows.
CSV parsing and schema statistics (host) are reported separately (`host_prep_s`).

`value`  — seconds per step with the parsed columns already resident in HBM.
`e2e`    — the same step through the public C-ABI with HOST columns: H2D of the
           parsed columns and D2H of A/N inside the timed region.
`roofline` — the matcher (kernel 6, the dominant kernel), algorithmic
           word-tests / its CUDA-event duration vs the measured LOP3 peak.
`cpu_baseline` — the reference (oracle/_ref: the reference's own C++ +
           restated mine/purify/infer) on this box's host cores, bounded sample.

`--impl reference` runs only the reference CPU path (rank 0) and prints its line.
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "IG fit seconds @148k NSL-KDD-shape; AND+POPC Gword/s vs int/HBM roofline"


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--rows", type=int, default=148517)
    ap.add_argument("--ratio", type=int, default=1, help="train tenths (1 = 10/90)")
    ap.add_argument("--seed", type=int, default=2507)
    ap.add_argument("--decimals", type=int, default=1)
    ap.add_argument("--cpu-sample-tests", type=int, default=400)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line).

    One `nvidia-smi -lms 200` child is started before the timed region and
    stopped after it, so no fork happens while steps are being issued."""

    def __init__(self):
        self.proc = None
        self.lines = []

    def start(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", os.environ.get("LOCAL_RANK", "0"), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.3)  # first sample lands before the timed region
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
            out, _ = self.proc.communicate()
        samples = [[x.strip() for x in ln.split(",")] for ln in out.splitlines() if ln.count(",") >= 5]
        if not samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(s[0]) for s in samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in samples for i in range(4) if s[2 + i].strip() == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(samples)}


def ncu_summary(path):
    """`traffic` (dram read+write bytes per launch) and pipe utilisation of the
    matcher from the committed `ncu --set full` capture of the same kernel."""
    import csv
    if not os.path.exists(path):
        return {}
    rows = list(csv.reader(open(path)))
    h, u, v = rows[0], rows[1], rows[2]
    get = {name: (float(v[i].replace(",", "")), u[i]) for i, name in enumerate(h)
           if name in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
                       "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
                       "smsp__issue_active.avg.pct_of_peak_sustained_active",
                       "lts__throughput.avg.pct_of_peak_sustained_elapsed",
                       "l1tex__throughput.avg.pct_of_peak_sustained_active")}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    try:
        traffic = sum(get[k][0] * scale.get(get[k][1], 1) for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        return {"traffic": traffic,
                "int_pipe_frac": get["sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"][0] / 100,
                "ncu": {"source": os.path.relpath(path, ROOT),
                        "alu_pipe_pct": get["sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"][0],
                        "issue_active_pct": get["smsp__issue_active.avg.pct_of_peak_sustained_active"][0],
                        "l2_throughput_pct": get["lts__throughput.avg.pct_of_peak_sustained_elapsed"][0],
                        "duration_ms_cold": get["gpu__time_duration.sum"][0],
                        "l1tex_throughput_pct": get.get("l1tex__throughput.avg.pct_of_peak_sustained_active",
                                                        (None,))[0],
                        "note": "L1 and issue bound: every lane loads a different posting word, and each AND "
                                "costs a shuffle, an address, a load and a vote besides its LOP3"}}
    except KeyError:
        return {}


def workload_config(args, n_train, n_test, extra=None):
    cfg = {"workload": f"synthetic NSL-KDD-shape {args.rows} records, {args.ratio * 10}/{100 - args.ratio * 10} "
                       f"train/test, p={args.decimals}",
           "records": args.rows, "train_rows": n_train, "test_rows": n_test, "seed": args.seed,
           "step": "tokenise+pack (train,test) + enumerate/dedup/support/score/purify + evidence(all test rows)",
           "l2": "inputs resident; working set (rows 1.7 MB, dictionaries ~0.3 GB) re-read every step"}
    if extra:
        cfg.update(extra)
    return cfg


def cpu_reference(csv: bytes, args, sample_tests: int):
    """Time the reference CPU path on this host; matcher on `sample_tests` rows,
    extrapolated linearly to all test rows (fused_score is linear in n_test)."""
    from oracle import ref
    if ref.available():
        kind = "reference"
        t0 = time.perf_counter()
        r = ref.run(csv, decimals=args.decimals, ratio_k=args.ratio, backend="parallel-cpu",
                    test_limit=sample_tests, stages=2)
        wall = time.perf_counter() - t0
        n_test_full = args.rows - args.ratio * args.rows // 10
        t = r.times
        scale = n_test_full / max(1, r.n_test)
        step = t["encode"] + t["enumerate"] + t["support"] + t["purify"] + (t["test_encode"] + t["match"]) * scale
        cores = ref.lib().igref_max_threads()
        sample = (f"full encode+fit ({r.n_train} train rows) + tokenise/match {r.n_test} of {n_test_full} test rows, "
                  f"matcher extrapolated x{scale:.1f}; wall {wall:.1f}s")
        return {"value": step, "unit": "s", "cores": cores, "kind": kind, "sample": sample,
                "phases_s": {k: round(v, 4) for k, v in t.items()}}
    # plain-C oracle port (no reference build on this box)
    import numpy as np
    from oracle import oracle
    from paper_2507_14222_b200 import api
    r = api.train_and_score(csv, decimals=args.decimals, ratio_k=args.ratio)
    Xa, Xn, T = r.train.matrix(0), r.train.matrix(1), r.test.matrix(2)
    t0 = time.perf_counter()
    f = oracle.fit(Xa, Xn)
    t1 = time.perf_counter()
    idx = np.arange(min(sample_tests, T.shape[0]))
    oracle.fused_score(f.pure[0].words, f.pure[0].scores, T[idx])
    oracle.fused_score(f.pure[1].words, f.pure[1].scores, T[idx])
    t2 = time.perf_counter()
    scale = T.shape[0] / max(1, len(idx))
    return {"value": (t1 - t0) + (t2 - t1) * scale, "unit": "s", "cores": os.cpu_count(), "kind": "port",
            "sample": f"oracle fit + matcher on {len(idx)} test rows x{scale:.1f}"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2507_14222_b200 import synth
    csv = synth.nsl_csv(args.rows, seed=args.seed)
    n_train = args.ratio * args.rows // 10
    vals = []
    for i in range(args.warmup + args.steps):
        # warm-up steps use a smaller matcher sample; timed steps the full bounded sample
        r = cpu_reference(csv, args, 8 if i < args.warmup else args.cpu_sample_tests)
        if i >= args.warmup:
            vals.append(r["value"])
    v = statistics.median(vals)
    line = {"metric": METRIC, "value": v, "unit": "s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": v * 1e3, "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": workload_config(args, n_train, args.rows - n_train), "impl": "reference",
            "cpu_baseline": {**{k: r[k] for k in ("unit", "cores", "kind", "sample")}, "value": v,
                             "steps_s": vals},
            "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_b200(args):
    import numpy as np
    import torch

    from paper_2507_14222_b200 import api, synth

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    # IG_BENCH_FORCE_SHARDED=1 (under torchrun) runs the sharded NCCL path even
    # at world size 1: a plumbing check of the N>1 code on a single GPU
    sharded_mode = world > 1 or os.environ.get("IG_BENCH_FORCE_SHARDED") == "1"
    out = sys.stdout
    if sharded_mode:
        # NCCL prints its banner on stdout at communicator creation: send fd 1
        # to stderr for the whole run and write the JSON line to the saved fd
        out = os.fdopen(os.dup(1), "w")
        sys.stdout.flush()
        os.dup2(2, 1)
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    t0 = time.perf_counter()
    csv = synth.nsl_csv(args.rows, seed=args.seed)
    t_gen = time.perf_counter() - t0

    ctx = api.Context(local)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)

    # host prep (not in the step): CSV parse, positional split, schema, typed columns
    t0 = time.perf_counter()
    table = api.read_csv(csv)
    n = table.rows
    n_train = args.ratio * n // 10
    tr, te = table.slice(0, n_train), table.slice(n_train, n)
    schema = api.infer_schema(tr, "label", decimals=args.decimals)
    cols_tr = api.Columns(tr, schema, True)
    cols_te = api.Columns(te, schema, False)
    host_prep = time.perf_counter() - t0
    n_test = cols_te.rows

    # resident copies for the `value` leg
    dev_tr = api.Columns(tr, schema, True).upload(ctx)
    dev_te = api.Columns(te, schema, False).upload(ctx)
    dA = torch.empty(n_test, dtype=torch.int64, device="cuda")
    dN = torch.empty(n_test, dtype=torch.int64, device="cuda")

    if sharded_mode:
        from paper_2507_14222_b200 import sharded
        ex = sharded.TorchExchange()

    def step_resident():
        enc = api.encode_training(dev_tr, ctx)
        if sharded_mode:
            # pair tiles round-robin, candidates to fingerprint owners (NCCL all-to-all),
            # owner-local support/coverage, partial evidence all-reduced.
            tenc = api.encode_rows(dev_te, enc, ctx)  # background pack + index during the fit
            res = sharded.fit_distributed(ctx, enc, rank, world, ex)
            a, n = sharded.evidence_distributed(res, tenc, ex)
            dA.copy_(a)
            dN.copy_(n)
            return enc, res.model, tenc
        # the test rows are packed and indexed in the background (index stream)
        # while the fit runs
        tenc = api.encode_rows(dev_te, enc, ctx)
        # fit + evidence: each class's matcher starts when its dictionary is ready
        model = api.fit_evidence_encoded(enc, tenc, d_A_ptr=dA.data_ptr(), d_N_ptr=dN.data_ptr())
        return enc, model, tenc

    def step_e2e():
        # both columns' H2D on the copy stream, training first: the training encode
        # waits for its 5 MB only, the test columns' 42 MB overlap the encode and fit
        cols_tr.prefetch(ctx)
        cols_te.prefetch(ctx)
        enc = api.encode_training(cols_tr, ctx)
        if sharded_mode:
            tenc = api.encode_rows(cols_te, enc, ctx)
            res = sharded.fit_distributed(ctx, enc, rank, world, ex)
            a, n = sharded.evidence_distributed(res, tenc, ex)
            return res.model, a.cpu().numpy(), n.cpu().numpy()
        tenc = api.encode_rows(cols_te, enc, ctx)  # from the prefetch: background pack + index
        return api.fit_evidence_encoded(enc, tenc)

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
            torch.cuda.synchronize()

    for _ in range(args.warmup):
        step_resident()
    barrier()

    # ---- value: resident inputs, CUDA events on the launching stream
    clocks = Clocks()
    clocks.start()
    launches0 = ctx.launches
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    barrier()
    gc.disable()
    for i in range(args.steps):
        enc = model = tenc = None  # release the previous step's results outside the timed window
        ev[i][0].record(stream)
        enc, model, tenc = step_resident()
        ev[i][1].record(stream)
    barrier()
    clk = clocks.stop()
    gc.enable()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    launches = (ctx.launches - launches0) / args.steps
    ms = statistics.median(step_ms)
    if dist is not None:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    phases = model.phase_ms()

    # ---- roofline of the dominant kernel: the matcher (kernel 6, grouped_scan<kMatch>)
    P = [model.count(0, 1), model.count(1, 1)]
    K = (tenc.logical_len + 63) // 64
    ctx.set_diagnostics(True)
    reps = 3
    for _ in range(reps):
        model.evidence_device(tenc.device_rows(2), n_test, dA.data_ptr(), dN.data_ptr())
    kms, words, nl = ctx.diag_match()
    ctx.set_diagnostics(False)
    lop3_s, popc_s = ctx.int_peaks()
    peak_words = lop3_s / 2 / 1e9   # a 64-bit word AND = 2 LOP3.32
    # the matcher's algorithmic work is W = (|P+| + |P-|) * n_test * K
    # word tests (the reference's dense (b & x) == b), per evidence call
    horiz = (P[0] + P[1]) * n_test * K
    launches_per_call = max(nl // reps, 1)
    ms_per_call = kms / reps
    achieved = horiz / (ms_per_call * 1e-3) / 1e9
    roofline = {"bound": "int", "kernel": "grouped_scan<kMatch> (matcher, kernel 6)", "achieved": achieved,
                "peak": peak_words, "unit": "Gword/s", "frac": achieved / peak_words, "traffic": None,
                "frac_is_effective": True,
                "algorithmic_work": (f"SURVEY.md §8(d) W = (|P+|+|P-|) * n_test * K = {horiz} 64-bit word tests per "
                                     f"evidence call ({launches_per_call} launches, {ms_per_call:.3f} ms)"),
                "note": ("W counts the dense (b & x) == b tests of the reference; the posting form skips almost all "
                         "of them, so W/t exceeds the LOP3 peak (an effective rate, SURVEY.md §8(d)).  The "
                         "hardware fraction is int_pipe_frac: the kernel's ALU-pipe utilisation measured by ncu."),
                "posting_word_ands": words // reps,
                "posting_word_and_rate_frac": (words / (kms * 1e-3) / 1e9) / peak_words,
                "peak_source": f"measured lop3 micro-kernel {lop3_s / 1e12:.2f} T LOP3.32/s (diag.cu)",
                "kernel_ms_per_launch": kms / max(nl, 1), "launches_per_step": launches_per_call,
                "share_of_step": ms_per_call / ms}
    roofline.update(ncu_summary(os.path.join(ROOT, "profiles", "r01_ncu_raw_grouped_scan_match.csv")))
    cfg_extra = {"L": tenc.logical_len, "K": K, "candidates": [model.count(0, 0), model.count(1, 0)], "pure": P}
    # release the resident leg's model before the e2e leg: at C4 it holds ~12 GB
    # and would force the memory pool to grow inside the e2e timed region
    enc = model = tenc = None
    gc.collect()
    torch.cuda.synchronize()

    # ---- e2e: host columns through the public ABI, H2D + D2H inside
    for _ in range(max(1, args.warmup // 2)):
        step_e2e()
    barrier()
    e2e_ms = []
    model_e = A = N = None
    gc.disable()
    for _ in range(args.steps):
        model_e = A = N = None
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        w0 = time.perf_counter()
        a.record(stream)
        model_e, A, N = step_e2e()
        b.record(stream)
        torch.cuda.synchronize()
        e2e_ms.append(max(a.elapsed_time(b), (time.perf_counter() - w0) * 1e3))
    gc.enable()
    e2e = statistics.median(e2e_ms)
    if dist is not None:
        t = torch.tensor([e2e], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e = float(t.item())
    h2d = cols_tr.nbytes + cols_te.nbytes
    d2h = 2 * n_test * 8

    # ---- csv leg (single GPU): CSV bytes on the host -> device ingest (parse,
    # schema, typed columns) -> encode -> fit -> evidence -> A/N on the host
    csv_leg = None
    if not sharded_mode:
        def step_csv():
            _, ctr_, cte_ = api.ingest_csv(csv, decimals=args.decimals, ratio_k=args.ratio, ctx=ctx)
            enc_ = api.encode_training(ctr_, ctx)
            tenc_ = api.encode_rows(cte_, enc_, ctx)
            return api.fit_evidence_encoded(enc_, tenc_)
        for _ in range(max(1, args.warmup // 2)):
            step_csv()
        csv_ms = []
        gc.disable()
        for _ in range(args.steps):
            torch.cuda.synchronize()
            w0 = time.perf_counter()
            step_csv()
            torch.cuda.synchronize()
            csv_ms.append((time.perf_counter() - w0) * 1e3)
        gc.enable()
        csv_leg = {"value": statistics.median(csv_ms) / 1e3, "unit": "s", "h2d_bytes_per_step": len(csv),
                   "d2h_bytes_per_step": d2h,
                   "note": "CSV bytes -> ig_ingest_csv (records, numbers, schema, columns on the GPU) -> encode -> "
                           "fit -> evidence -> A/N; the host parse this replaces is host_prep_s"}

    # ---- SURVEY.md §8(d) "fit seconds": H2D of the parsed training columns ->
    # tokenise -> enumerate / dedup / support / score / purify -> the pure
    # dictionaries (patterns, supports, scores) on the host; and the matcher
    # alone (resident test encoding -> A/N on the host), as separate numbers
    fit_leg = None
    if not sharded_mode:
        dev_tenc = api.encode_rows(dev_te, api.encode_training(dev_tr, ctx), ctx)

        def step_fit():
            enc_ = api.encode_training(cols_tr, ctx)
            model_ = api.fit_encoded(enc_)
            return model_, [model_.dictionary(c, 1) for c in range(2)]

        def step_match(model_):
            return model_.evidence_encoded(dev_tenc)

        for _ in range(max(1, args.warmup // 2)):
            m_, _ = step_fit()
            step_match(m_)
        fit_ms, match_ms, dict_bytes = [], [], 0
        gc.disable()
        for _ in range(args.steps):
            m_ = dicts = None  # the previous dictionaries' host blocks return to the pool
            torch.cuda.synchronize()
            w0 = time.perf_counter()
            m_, dicts = step_fit()
            torch.cuda.synchronize()
            w1 = time.perf_counter()
            step_match(m_)
            torch.cuda.synchronize()
            w2 = time.perf_counter()
            fit_ms.append((w1 - w0) * 1e3)
            match_ms.append((w2 - w1) * 1e3)
            dict_bytes = sum(d.words.nbytes + d.supports.nbytes + d.scores.nbytes for d in dicts)
        gc.enable()
        m_ = dicts = None
        fit_leg = {"fit_s": statistics.median(fit_ms) / 1e3, "matcher_s": statistics.median(match_ms) / 1e3,
                   "unit": "s", "h2d_bytes_per_step": cols_tr.nbytes, "d2h_bytes_per_step": dict_bytes,
                   "note": "fit: parsed training columns (host) -> encode -> fit -> both pure dictionaries copied "
                           "to the host (into page-locked arrays from the library's host pool, reused across fits "
                           "once freed); matcher: resident test encoding -> A/N on the host"}


    line = {"metric": METRIC, "value": ms / 1e3, "unit": "s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": workload_config(args, n_train, n_test, {"parallelism": (f"sharded{world}: pair tiles round-robin, NCCL all-to-all to fingerprint owners, "
                                                                              "all-reduce of partial evidence") if sharded_mode else "1gpu",
                                                              **cfg_extra}),
            "phases_ms": {"fit": phases, "step_median": ms, "steps": step_ms},
            "host_prep_s": host_prep, "gen_s": t_gen,
            "e2e": {"value": e2e / 1e3, "unit": "s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "e2e_csv": csv_leg,
            "fit_and_matcher": fit_leg,
            "gpu_launches": launches, "clocks": clk, "roofline": roofline}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_reference(csv, args, args.cpu_sample_tests)
    if rank == 0:
        print(json.dumps(line), file=out, flush=True)
    if dist is not None:
        dist.destroy_process_group()


def _all_host_threads():
    """The CPU reference (oracle/_ref, OpenMP) runs with every host thread this
    process may use.  torch.distributed.run exports OMP_NUM_THREADS=1 to each
    rank, which would time the reference arm single-threaded under torchrun;
    libgomp reads the variable when oracle/_ref is loaded, so set it first."""
    try:
        n = len(os.sched_getaffinity(0))
    except AttributeError:
        n = os.cpu_count() or 1
    os.environ["OMP_NUM_THREADS"] = str(n)


def main():
    args = parse_args()
    _all_host_threads()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
