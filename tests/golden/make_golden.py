"""Generate the golden fixtures under tests/golden/ from the reference itself.

Run here (where /root/reference exists):  python tests/golden/make_golden.py

Every value below is produced by oracle/_ref/libigref.so, i.e. the reference's
own compiled C++ (proj/src/{bitpack,csv,kernels,pipeline}.cpp) plus the
restated mine/purify/infer modules (oracle/ref_shim.cpp).  The fixtures pin the
plain-C oracle and the Python pipeline restatement (tests/test_oracle_golden.py)
and are the known answers the CUDA path is compared with on the GPU box, where
/root/reference is absent.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402
from paper_2507_14222_b200 import synth  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def pack(bits, L):
    k = (L + 63) // 64
    w = np.zeros(k, np.uint64)
    for b in bits:
        w[b // 64] |= np.uint64(1) << np.uint64(b % 64)
    return w.view(np.int64)


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode() + str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def running_example():
    # tokens a..e are bits 0..4, L = 5.
    a, b, c, d, e = range(5)
    L = 5
    Xp = np.stack([pack(s, L) for s in ([a, b, c], [a, b, d], [a, c, d])])
    Xn = np.stack([pack(s, L) for s in ([a, b, e], [c, d, e])])
    cand_p = ref.mine(Xp, L, backend="reference", threads=1)
    cand_n = ref.mine(Xn, L, backend="reference", threads=1)
    keep_p = ref.coverage_any(cand_p.words, L, Xn, L, backend="reference") == 0
    keep_n = ref.coverage_any(cand_n.words, L, Xp, L, backend="reference") == 0
    probes = np.stack([pack(s, L) for s in ([a, c, d, e], [a, b, e], [b])])
    A = ref.fused_score(cand_p.words[keep_p], L, cand_p.scores[keep_p], probes, L, backend="reference")
    N = ref.fused_score(cand_n.words[keep_n], L, cand_n.scores[keep_n], probes, L, backend="reference")
    win = ref.pair_intersect_batch(Xp, L, 0, 1, 3, backend="reference")
    return dict(
        L=L, attack=Xp.tolist(), normal=Xn.tolist(),
        cand_attack=dict(words=cand_p.words.tolist(), supports=cand_p.supports.tolist(), scores=cand_p.scores.tolist()),
        cand_normal=dict(words=cand_n.words.tolist(), supports=cand_n.supports.tolist(), scores=cand_n.scores.tolist()),
        pure_attack_mask=keep_p.astype(int).tolist(), pure_normal_mask=keep_n.astype(int).tolist(),
        probes=probes.tolist(), A=A.tolist(), N=N.tolist(), pair_window_0_1_3=win.tolist(),
    )


def random_mine(count=40, seed=11):
    rng = np.random.default_rng(seed)
    cases = {}
    for i in range(count):
        L = int(rng.choice([1, 5, 63, 64, 65, 96, 130]))
        k = (L + 63) // 64
        n_a, n_n, n_t = (int(x) for x in rng.integers(1, 48, 3))
        dens = float(rng.uniform(0.2, 0.9))

        def rows(n):
            bits = rng.random((n, L)) < dens
            out = np.zeros((n, k), np.uint64)
            for j in range(L):
                out[:, j // 64] |= bits[:, j].astype(np.uint64) << np.uint64(j % 64)
            return out.view(np.int64)

        Xa, Xn, T = rows(n_a), rows(n_n), rows(n_t)
        ca = ref.mine(Xa, L, pair_batch=int(rng.integers(1, 9)), backend="reference", threads=1)
        cn = ref.mine(Xn, L, backend="parallel-cpu", threads=3)
        ka = ref.coverage_any(ca.words, L, Xn, L) == 0
        kn = ref.coverage_any(cn.words, L, Xa, L) == 0
        A = ref.fused_score(ca.words[ka], L, ca.scores[ka], T, L)
        N = ref.fused_score(cn.words[kn], L, cn.scores[kn], T, L)
        pre = f"c{i}_"
        cases.update({pre + "L": np.array(L), pre + "attack": Xa, pre + "normal": Xn, pre + "tests": T,
                      pre + "ca_words": ca.words, pre + "ca_sup": ca.supports, pre + "ca_sc": ca.scores,
                      pre + "cn_words": cn.words, pre + "cn_sup": cn.supports, pre + "cn_sc": cn.scores,
                      pre + "keep_a": ka.astype(np.uint8), pre + "keep_n": kn.astype(np.uint8),
                      pre + "A": A, pre + "N": N})
    np.savez_compressed(os.path.join(OUT, "random_mine.npz"), count=np.array(count), **cases)


ZPROBES = [(0.05, 1), (-0.05, 1), (0.15, 1), (0.25, 1), (-0.04, 1), (1e19, 1), (-1e19, 2), (1.45, 1),
           (2.675, 2), (-2.675, 2), (0.0, 0), (-0.0, 3), (0.5, 0), (-0.5, 0), (1.5, 0), (2.5, 0),
           (123.456789, 4), (-1.2247448713915890, 2), (1e-7, 6), (4.5e18, 1), (8.99e17, 1), (3.14159, 12)]

FUZZ_CSV = (
    "﻿a,b,c,label\r\n"
    "1,tcp,\"x,y\",normal\n"
    "2,udp,,neptune\r"
    "3,,\"q\"\"q\",normal\n"
    "+5,tcp,z,normal\n"
    "1e3,icmp,z,smurf\n"
    ".5,tcp,x,normal\n"
    "1,tcp,\"x,y\",neptune\n"
    "7,tcp,\"multi\nline\",neptune\n"
).encode()

NUM_CSV = (
    "f0,f1,f2,f3,label\n"
    "1,5,0.10,7,normal\n"
    "2,5,0.20,,attack\n"
    "3,5,0.15,-7,normal\n"
    "1,5,0.25,1e2,attack\n"
    "1,5,0.35,7,attack\n"
    "2,5,-0.05,7,normal\n"
    "2,5,0.05,3,attack\n"
).encode()


def tokenizer():
    z = [dict(z=zv, p=p, s=ref.format_zscore(zv, p)) for zv, p in ZPROBES]
    runs = {}
    for name, csv, label, dec, ntr in (("fuzz", FUZZ_CSV, "label", 1, 7), ("num", NUM_CSV, "label", 1, 5),
                                       ("num_p2", NUM_CSV, "label", 2, 6), ("num_p0", NUM_CSV, "label", 0, 7)):
        r = ref.run(csv, label_col=label, decimals=dec, train_rows=ntr, stages=0)
        runs[name] = dict(csv=csv.decode("utf-8"), decimals=dec, train_rows=ntr, L=r.L, vocab=r.vocab,
                          attack=r.attack.tolist(), normal=r.normal.tolist(),
                          removed=[int(x) for x in r.removed_rows], kind=r.kind.tolist(),
                          mean=r.mean.tolist(), std=r.std.tolist())
    return dict(zscore=z, runs=runs)


def nsl_digest():
    """C1: synthetic NSL-shape 2,000 records, p=1, 80/20 — the CPU-oracle config."""
    csv = synth.nsl_csv(2000, seed=2507)
    r = ref.run(csv, decimals=1, ratio_k=8, backend="parallel-cpu")
    out = dict(rows=2000, seed=2507, decimals=1, ratio_k=8, L=r.L, n_attack=int(r.attack.shape[0]),
               n_normal=int(r.normal.shape[0]), n_test=int(r.tests.shape[0]),
               csv_sha256=hashlib.sha256(csv).hexdigest(),
               vocab_sha256=hashlib.sha256("\n".join(r.vocab).encode()).hexdigest(),
               rows_digest=digest(r.attack, r.normal, r.tests),
               cand_counts=[int(c[0].shape[0]) for c in r.cand], pure_counts=[int(p[0].shape[0]) for p in r.pure],
               cand_digest=[digest(*c) for c in r.cand], pure_digest=[digest(*p) for p in r.pure],
               A_digest=digest(r.A), N_digest=digest(r.N), A_sum=int(r.A.sum()), N_sum=int(r.N.sum()),
               labels_digest=digest(r.labels), regulation_digest=digest(r.regulation),
               mu=r.mu, sigma=r.sigma)
    return out


def main():
    if not ref.available():
        raise SystemExit("build oracle/_ref first: make -C oracle ref")
    with open(os.path.join(OUT, "spec_examples.json"), "w") as f:
        json.dump(running_example(), f, indent=1)
    random_mine()
    with open(os.path.join(OUT, "tokenizer.json"), "w") as f:
        json.dump(tokenizer(), f, indent=1)
    with open(os.path.join(OUT, "nsl_c1.json"), "w") as f:
        json.dump(nsl_digest(), f, indent=1)
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
