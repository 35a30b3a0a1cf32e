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
`roofline` — per hot kernel (pair_enum, support, cover, matcher): exact useful
           64-bit word-ANDs / CUDA-event kernel time vs the measured LOP3 peak,
           from one extra step with the classes serialised; the top-level entry
           is the kernel with the most time (the matcher).
`scale_leg` — BASELINE.json configs[3] (the same records at 80/20), timed like
           `value`: the strong-scaling number of the driver's N-GPU runs.
`cpu_baseline` — the reference (oracle/_ref: the reference's own C++ +
           restated mine/purify/infer) on this box's host cores: full fit, a
           bounded slice of the matcher scaled to all test rows.

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
    ap.add_argument("--scale-ratio", type=int, default=8, help="train tenths of the scale leg (0 = off)")
    ap.add_argument("--cpu-sample-tests", type=int, default=2000)
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


def ncu_summary(path, launches=1):
    """`traffic` (DRAM read + write bytes per launch) and pipe utilisation from
    the committed `ncu --set full` capture of the same kernel (one launch)."""
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
    tscale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}
    try:
        traffic = sum(get[k][0] * scale.get(get[k][1], 1) for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        return {"traffic": traffic,
                "ncu": {"source": os.path.relpath(path, ROOT),
                        "alu_pipe_pct": get["sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"][0],
                        "issue_active_pct": get["smsp__issue_active.avg.pct_of_peak_sustained_active"][0],
                        "l2_throughput_pct": get["lts__throughput.avg.pct_of_peak_sustained_elapsed"][0],
                        "l1tex_throughput_pct": get.get("l1tex__throughput.avg.pct_of_peak_sustained_active",
                                                        (None,))[0],
                        "duration_ms_cold": get["gpu__time_duration.sum"][0] *
                        tscale.get(get["gpu__time_duration.sum"][1], 1.0)}}
    except KeyError:
        return {}


KERNEL_INFO = {
    "pair_enum": ("pair_enum (kernels 2+3: pair AND + fingerprint + tile/device dedup)",
                  "SURVEY.md §8(d) (2): K word-ANDs per pair u <= v of the class's distinct canonical rows",
                  "r02_ncu_raw_pair_enum.csv"),
    "support": ("half_scan<kSupport> (kernel 5: f_c(b) by posting AND + POPC, two short-list patterns per warp)",
                "posting word-ANDs on live list words (counted exactly by a counting re-run)",
                "r02_ncu_raw_half_scan_support.csv"),
    "cover": ("half_scan<kCover> (kernel 4: opposite-class subset filter, vote early exit, two short-list "
              "patterns per warp)",
              "posting word-ANDs on live list words up to the first covering word (counted exactly)",
              "r02_ncu_raw_half_scan_cover.csv"),
    "match": ("grouped_scan<kMatch> (kernel 6: matcher, difference-array runs)",
              "posting word-ANDs on live list words (counted exactly)",
              "r02_ncu_raw_grouped_scan_match.csv"),
}


def kernel_rooflines(diag, peak_words, lop3_s, step_ms, horiz):
    """achieved = useful 64-bit word-ANDs / kernel time against
    the measured LOP3 peak (2 LOP3.32 per word-AND).  The useful work is what
    the kernel actually performs (the posting form skips the reference's dense
    (b & x) == b tests; that dense W is kept only as `effective_rate`)."""
    kernels = []
    for name, (label, work_def, ncu_file) in KERNEL_INFO.items():
        kms, work, nl = diag[name]
        if nl == 0 or kms <= 0:
            continue
        achieved = work / (kms * 1e-3) / 1e9
        e = {"kernel": label, "id": name, "launches_per_step": nl, "ms_per_step": kms,
             "ms_per_launch": kms / nl, "useful_word_ands_per_step": work, "work_definition": work_def,
             "achieved": achieved, "peak": peak_words, "unit": "Gword/s", "frac": achieved / peak_words,
             "share_of_step": kms / step_ms}
        e.update(ncu_summary(os.path.join(ROOT, "profiles", ncu_file), nl))
        kernels.append(e)
    top = max(kernels, key=lambda e: e["ms_per_step"])
    out = {"bound": "int", "kernel": top["kernel"], "achieved": top["achieved"], "peak": peak_words,
           "unit": "Gword/s", "frac": top["frac"], "traffic": top.get("traffic"),
           "peak_source": f"measured LOP3 micro-kernel {lop3_s / 1e12:.2f} T LOP3.32/s (diag.cu) / 2 per 64-bit AND",
           "timing": "one extra step with diagnostics on: classes serialised, CUDA events around each hot launch "
                     "on its stream; work from a counting re-run of the same launch",
           "kernels": kernels}
    m = diag["match"]
    if m[2]:
        out["effective_rate"] = {
            "kernel": "matcher", "dense_word_tests_per_step": horiz, "Gword_per_s": horiz / (m[0] * 1e-3) / 1e9,
            "note": "SURVEY.md §8(d) (6) W = (|P+|+|P-|) * n_test * K, the reference's dense (b & x) == b word "
                    "tests, over the matcher's time: an effective rate, not a hardware fraction"}
    return out


def workload_config(args, n_train, n_test, extra=None):
    cfg = {"workload": f"synthetic NSL-KDD-shape {args.rows} records, {args.ratio * 10}/{100 - args.ratio * 10} "
                       f"train/test, p={args.decimals}",
           "records": args.rows, "train_rows": n_train, "test_rows": n_test, "seed": args.seed,
           "step": "tokenise+pack (train,test) + enumerate/dedup/support/score/purify + evidence(all test rows)",
           "l2": "inputs resident; working set (rows 1.7 MB, dictionaries ~0.3 GB) re-read every step"}
    if extra:
        cfg.update(extra)
    return cfg


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_reference(csv: bytes, args, sample_tests: int, step: int = 0):
    """One step of the reference's own CPU path (oracle/_ref: proj/src/*.cpp
    compiled by oracle/Makefile + the restated mine/purify/infer) on this host,
    every host thread: encode + full fit of all training rows, then tokenise +
    match a bounded slice of the test rows, [step * S, (step + 1) * S) mod
    n_test, so successive steps measure different parts of the test set.  The
    matcher is linear in the test rows (one independent fused_score per row,
    kernels.cpp:156-178), so the full step is the fit plus the slice's matcher
    time scaled to all test rows.  No fallback: the reference must be built."""
    from oracle import ref
    if not ref.available():
        raise SystemExit("oracle/_ref/libigref.so missing: build it with `make -C oracle ref` where "
                         "/root/reference exists (it ships to the GPU box in the snapshot)")
    n_test_full = args.rows - args.ratio * args.rows // 10
    S = max(1, min(sample_tests, n_test_full))
    off = (step * S) % n_test_full
    t0 = time.perf_counter()
    r = ref.run(csv, decimals=args.decimals, ratio_k=args.ratio, backend="parallel-cpu",
                test_offset=off, test_limit=S, stages=2)
    wall = time.perf_counter() - t0
    t = r.times
    scale = n_test_full / max(1, r.n_test)
    full = t["encode"] + t["enumerate"] + t["support"] + t["purify"] + (t["test_encode"] + t["match"]) * scale
    cores = ref.lib().igref_max_threads()
    return {"value": full, "unit": "s", "cores": cores, "kind": "reference", "wall_s": wall,
            "sample": (f"encode + full fit of all {r.n_train} training rows, then tokenise + match test rows "
                       f"[{off}, {off + r.n_test}) of {n_test_full} (matcher scaled x{scale:.2f} to all test rows)"),
            "cpu": cpu_model(), "isa": "oracle/_ref built -march=x86-64-v3 (AVX2, FMA, POPCNT)",
            "phases_s": {k: round(v, 4) for k, v in t.items()}, "matched_rows": int(r.n_test)}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2507_14222_b200 import synth
    csv = synth.nsl_csv(args.rows, seed=args.seed)
    n_train = args.ratio * args.rows // 10
    n_test = args.rows - n_train
    # warm-up: the reference on the first 2,000 records (thread pool, page cache, allocator)
    small = b"\n".join(csv.split(b"\n")[:2001]) + b"\n"
    for _ in range(args.warmup):
        from oracle import ref
        ref.run(small, decimals=args.decimals, ratio_k=8, backend="parallel-cpu")
    vals, walls, matched = [], [], 0
    for i in range(args.steps):
        r = cpu_reference(csv, args, args.cpu_sample_tests, step=i)
        vals.append(r["value"])
        walls.append(r["wall_s"])
        matched += r["matched_rows"]
    v = statistics.median(vals)
    line = {"metric": METRIC, "value": v, "unit": "s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": statistics.median(walls) * 1e3, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": workload_config(args, n_train, n_test), "impl": "reference",
            "value_definition": ("full C3 step time: encode + fit measured in full every step, the matcher measured "
                                 "on a rotating slice of the test rows and scaled linearly; ms_per_step is the "
                                 "measured wall time of one such step"),
            "cpu_baseline": {**{k: r[k] for k in ("unit", "cores", "kind", "cpu", "isa")}, "value": v,
                             "sample": (f"{args.steps} steps, each encode + full fit + a {args.cpu_sample_tests}-row "
                                        f"test slice (rotating; {matched} of {n_test} test rows matched over the run)"),
                             "steps_s": vals, "steps_wall_s": walls},
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

    # ---- roofline, per hot kernel: one more step with diagnostics on (classes
    # one after the other, every hot launch timed with CUDA events on its own
    # stream, then re-run in a counting variant for its exact useful work)
    P = [model.count(0, 1), model.count(1, 1)]
    K = (tenc.logical_len + 63) // 64
    horiz = (P[0] + P[1]) * n_test * K  # dense word tests of the reference
    enc = model = tenc = None
    ctx.set_diagnostics(True)
    torch.cuda.synchronize()
    enc, model, tenc = step_resident()
    torch.cuda.synchronize()
    diag = {name: ctx.diag_kernel(name) for name in api.Context.DIAG_KERNELS}
    ctx.set_diagnostics(False)
    lop3_s, popc_s = ctx.int_peaks()
    peak_words = lop3_s / 2 / 1e9   # a 64-bit word AND = 2 LOP3.32 (measured micro-kernel, diag.cu)
    roofline = kernel_rooflines(diag, peak_words, lop3_s, ms, horiz)
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
        # the CSV bytes in page-locked host memory, like the e2e columns
        import numpy as np
        csv_pinned = api.pinned_array(len(csv), np.uint8)
        csv_pinned[:] = np.frombuffer(csv, np.uint8)

        def step_csv():
            _, ctr_, cte_ = api.ingest_csv(csv_pinned, decimals=args.decimals, ratio_k=args.ratio, ctx=ctx)
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
                   "note": "CSV bytes (page-locked host buffer) -> ig_ingest_csv (records, numbers, schema, columns on "
                           "the GPU) -> encode -> fit -> evidence -> A/N; the host parse this replaces is host_prep_s"}

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

    # ---- scale leg: BASELINE.json configs[3] (C4: the same 148,517 records at
    # 80/20, 118,813 training rows), the strong-scaling configuration of the
    # driver's N-GPU runs; resident columns, fit + evidence per step, timed like
    # `value` (CUDA events, max over ranks).  At N > 1 the sharded path.
    scale_leg = None
    if args.scale_ratio and args.scale_ratio != args.ratio:
        enc = model = tenc = None
        gc.collect()
        ntr4 = args.scale_ratio * n // 10
        tr4, te4 = table.slice(0, ntr4), table.slice(ntr4, n)
        schema4 = api.infer_schema(tr4, "label", decimals=args.decimals)
        d_tr4 = api.Columns(tr4, schema4, True).upload(ctx)
        d_te4 = api.Columns(te4, schema4, False).upload(ctx)
        n_te4 = d_te4.rows
        dA4 = torch.empty(n_te4, dtype=torch.int64, device="cuda")
        dN4 = torch.empty(n_te4, dtype=torch.int64, device="cuda")

        def step_scale():
            enc_ = api.encode_training(d_tr4, ctx)
            tenc_ = api.encode_rows(d_te4, enc_, ctx)
            if sharded_mode:
                res_ = sharded.fit_distributed(ctx, enc_, rank, world, ex)
                a_, n_ = sharded.evidence_distributed(res_, tenc_, ex)
                dA4.copy_(a_)
                dN4.copy_(n_)
                return res_.model
            return api.fit_evidence_encoded(enc_, tenc_, d_A_ptr=dA4.data_ptr(), d_N_ptr=dN4.data_ptr())

        m4 = step_scale()
        m4 = None
        barrier()
        sc_steps = max(3, min(args.steps, 10))
        ev4 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(sc_steps)]
        gc.disable()
        for i in range(sc_steps):
            m4 = None
            ev4[i][0].record(stream)
            m4 = step_scale()
            ev4[i][1].record(stream)
        barrier()
        gc.enable()
        sc_ms_all = [a.elapsed_time(b) for a, b in ev4]
        sc_ms = statistics.median(sc_ms_all)
        if dist is not None:
            t = torch.tensor([sc_ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            sc_ms = float(t.item())
        scale_leg = {"config": {"workload": f"synthetic NSL-KDD-shape {n} records, {args.scale_ratio * 10}/"
                                            f"{100 - args.scale_ratio * 10} train/test, p={args.decimals} "
                                            "(BASELINE.json configs[3])",
                                "train_rows": ntr4, "test_rows": n_te4,
                                "candidates": [m4.count(0, 0), m4.count(1, 0)] if not sharded_mode else None,
                                "pure": [m4.count(0, 1), m4.count(1, 1)] if not sharded_mode else None},
                     "value": sc_ms / 1e3, "unit": "s", "ms_per_step": sc_ms, "steps": sc_steps, "steps_ms": sc_ms_all,
                     "n_gpus": world, "scaling": "strong",
                     "note": "resident columns; encode + fit + evidence of all test rows per step; the number the "
                             "1/2/4/8-GPU strong-scaling efficiency of configs[3] is read from"}
        m4 = d_tr4 = d_te4 = None
        gc.collect()

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
            "scale_leg": scale_leg,
            "gpu_launches": launches, "clocks": clk, "roofline": roofline}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_reference(csv, args, args.cpu_sample_tests)
        line["cpu_baseline"]["sample"] += "; one step"
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
