"""Matcher experiments at C3: times model.evidence_device under different env switches."""
import os, sys, json, time, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 1 and sys.argv[1] == "child":
    import torch
    from paper_2507_14222_b200 import api, synth
    csv = synth.nsl_csv(148517, seed=2507)
    ctx = api.Context(0)
    st = torch.cuda.current_stream(); ctx.set_stream(st.cuda_stream)
    r = api.train_and_score(csv, decimals=1, ratio_k=1, ctx=ctx)
    n = r.test.rows(2)
    dA = torch.empty(n, dtype=torch.int64, device="cuda"); dN = torch.empty_like(dA)
    ts = []
    for i in range(4):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st); r.model.evidence_device(r.test.device_rows(2), n, dA.data_ptr(), dN.data_ptr()); b.record(st)
        torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    ok = bool((dA.cpu().numpy() == r.A).all() and (dN.cpu().numpy() == r.N).all())
    ctx.set_diagnostics(True); r.model.evidence_device(r.test.device_rows(2), n, dA.data_ptr(), dN.data_ptr()); dm = ctx.diag_match()
    print(json.dumps({"env": {k: v[-30:] for k, v in os.environ.items() if k.startswith("IG_")}, "ms": ts, "diag": dm, "same_as_first": ok}))
    sys.exit(0)
for env in ({}, {"IG_B200_LIB": os.path.join(os.path.dirname(os.path.abspath(__file__)), "libig_b200_nohits.so")}):
    e = dict(os.environ); e.update(env)
    out = subprocess.run([sys.executable, __file__, "child"], env=e, capture_output=True, text=True)
    print(out.stdout.strip() or out.stderr[-2000:], flush=True)
