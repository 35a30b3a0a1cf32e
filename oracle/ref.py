"""ctypes driver for oracle/_ref/libigref.so — TEST INFRASTRUCTURE ONLY.

`_ref` is the reference's own C++ (proj/src/*.cpp) compiled by oracle/Makefile
plus oracle/ref_shim.cpp (the missing mine/purify/infer modules restated on the
reference's types).  Only tests/, __graft_entry__.smoke() and bench.py's
reference / cpu_baseline legs may import this module.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libigref.so")
REF_B200_SO = os.path.join(HERE, "_ref", "libigref_b200.so")  # + integration/ shim on libig_b200.so

STATUS = {1: ValueError, 2: IndexError, 3: "ConfigError", 4: OSError, 5: "DataError",
          6: "ArithmeticError", 7: RuntimeError}


class RefError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"[{status}] {msg}")
        self.status = status
        self.msg = msg


_libs = {}


def available(b200: bool = False) -> bool:
    return os.path.exists(REF_B200_SO if b200 else REF_SO)


def lib(b200: bool = False):
    key = bool(b200)
    if key not in _libs:
        path = REF_B200_SO if b200 else REF_SO
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (make -C oracle ref / refb200)")
        L = C.CDLL(path)
        p64 = C.POINTER(C.c_int64)
        sz = C.c_size_t
        L.igref_last_error.restype = C.c_char_p
        L.igref_max_threads.restype = C.c_int
        L.igref_format_zscore.argtypes = [C.c_double, C.c_int, C.c_char_p, sz]
        L.igref_pair_intersect_batch.argtypes = [C.c_char_p, C.c_int, p64, sz, C.c_uint32, sz, sz, sz, p64]
        L.igref_coverage_any.argtypes = [C.c_char_p, C.c_int, p64, sz, C.c_uint32, p64, sz, C.c_uint32, sz,
                                         C.POINTER(C.c_uint8)]
        L.igref_fused_score.argtypes = [C.c_char_p, C.c_int, p64, sz, C.c_uint32, p64, sz, p64, sz,
                                        C.c_uint32, p64]
        L.igref_enumerate.argtypes = [C.c_char_p, C.c_int, sz, p64, sz, C.c_uint32, C.POINTER(C.c_void_p)]
        L.igref_cand_free.argtypes = [C.c_void_p]
        L.igref_cand_count.argtypes = [C.c_void_p]
        L.igref_cand_count.restype = sz
        for f in ("igref_cand_words", "igref_cand_supports", "igref_cand_scores"):
            getattr(L, f).argtypes = [C.c_void_p]
            getattr(L, f).restype = p64
        L.igref_count_support.argtypes = [C.c_void_p, C.c_int, p64, sz, C.c_uint32]
        L.igref_score_patterns.argtypes = [C.c_void_p]
        L.igref_total_score.argtypes = [p64, sz, p64]
        L.igref_run_create.argtypes = [C.c_char_p, sz, C.c_char_p, C.c_char_p, C.c_char_p, C.c_int, C.c_int,
                                       sz, C.c_char_p, C.c_int, sz, sz, sz, sz, C.c_int, C.c_double,
                                       C.POINTER(C.c_void_p)]
        L.igref_run_free.argtypes = [C.c_void_p]
        L.igref_run_L.argtypes = [C.c_void_p]
        L.igref_run_L.restype = C.c_uint32
        L.igref_run_vocab.argtypes = [C.c_void_p]
        L.igref_run_vocab.restype = C.c_char_p
        L.igref_run_rows.argtypes = [C.c_void_p, C.c_int]
        L.igref_run_rows.restype = sz
        L.igref_run_matrix.argtypes = [C.c_void_p, C.c_int]
        L.igref_run_matrix.restype = p64
        L.igref_run_removed.argtypes = [C.c_void_p]
        L.igref_run_removed.restype = C.POINTER(C.c_uint64)
        L.igref_run_dict_count.argtypes = [C.c_void_p, C.c_int]
        L.igref_run_dict_count.restype = sz
        L.igref_run_dict.argtypes = [C.c_void_p, C.c_int, C.c_int]
        L.igref_run_dict.restype = p64
        L.igref_run_evidence.argtypes = [C.c_void_p, C.c_int]
        L.igref_run_evidence.restype = p64
        L.igref_run_labels.argtypes = [C.c_void_p, C.c_int]
        L.igref_run_labels.restype = C.POINTER(C.c_uint8)
        L.igref_run_stats.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.igref_run_times.argtypes = [C.c_void_p]
        L.igref_run_times.restype = C.POINTER(C.c_double)
        L.igref_run_cols.argtypes = [C.c_void_p]
        L.igref_run_cols.restype = sz
        L.igref_run_schema.argtypes = [C.c_void_p, C.POINTER(C.c_uint8), C.POINTER(C.c_double),
                                       C.POINTER(C.c_double), C.POINTER(C.c_size_t)]
        _libs[key] = L
    return _libs[key]


def _check(status: int, b200: bool = False):
    if status:
        raise RefError(status, lib(b200).igref_last_error().decode())


def _p64(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_int64))


def _words(a: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


def format_zscore(z: float, decimals: int) -> str:
    buf = C.create_string_buffer(64)
    _check(lib().igref_format_zscore(z, decimals, buf, 64))
    return buf.value.decode()


def pair_intersect_batch(rows: np.ndarray, L: int, left: int, jb: int, je: int,
                         backend: str = "reference", threads: int = 0) -> np.ndarray:
    rows = _words(rows)
    k = (L + 63) // 64
    out = np.zeros((max(je - jb, 0), k), np.int64)
    b = backend == "b200"
    _check(lib(b).igref_pair_intersect_batch(backend.encode(), threads, _p64(rows), rows.shape[0], L,
                                             left, jb, je, _p64(out)), b)
    return out


def coverage_any(pat: np.ndarray, Lp: int, opp: np.ndarray, Lo: int, block: int = 4096,
                 backend: str = "parallel-cpu", threads: int = 0) -> np.ndarray:
    pat, opp = _words(pat), _words(opp)
    mask = np.zeros(pat.shape[0], np.uint8)
    b = backend == "b200"
    _check(lib(b).igref_coverage_any(backend.encode(), threads, _p64(pat), pat.shape[0], Lp, _p64(opp),
                                     opp.shape[0], Lo, block, mask.ctypes.data_as(C.POINTER(C.c_uint8))), b)
    return mask


def fused_score(pat: np.ndarray, Lp: int, scores: np.ndarray, tests: np.ndarray, Lt: int,
                backend: str = "parallel-cpu", threads: int = 0) -> np.ndarray:
    pat, tests = _words(pat), _words(tests)
    scores = np.ascontiguousarray(scores, np.int64)
    out = np.zeros(tests.shape[0], np.int64)
    b = backend == "b200"
    _check(lib(b).igref_fused_score(backend.encode(), threads, _p64(pat), pat.shape[0], Lp, _p64(scores),
                                    scores.shape[0], _p64(tests), tests.shape[0], Lt, _p64(out)), b)
    return out


@dataclass
class Candidates:
    words: np.ndarray
    supports: np.ndarray | None = None
    scores: np.ndarray | None = None


def mine(rows: np.ndarray, L: int, pair_batch: int = 8192, backend: str = "reference",
         threads: int = 0, support: bool = True) -> Candidates:
    """enumerate_candidates → count_support → score_patterns (mine.hpp:38-48)."""
    rows = _words(rows)
    b200 = backend == "b200"
    h = C.c_void_p()
    _check(lib(b200).igref_enumerate(backend.encode(), threads, pair_batch, _p64(rows), rows.shape[0], L,
                                 C.byref(h)), b200)
    try:
        n = lib(b200).igref_cand_count(h)
        k = (L + 63) // 64
        words = np.ctypeslib.as_array(lib(b200).igref_cand_words(h), (n * k,)).reshape(n, k).copy() if n else \
            np.zeros((0, k), np.int64)
        if not support:
            return Candidates(words)
        _check(lib(b200).igref_count_support(h, threads, _p64(rows), rows.shape[0], L), b200)
        _check(lib(b200).igref_score_patterns(h), b200)
        sup = np.ctypeslib.as_array(lib(b200).igref_cand_supports(h), (n,)).copy() if n else np.zeros(0, np.int64)
        sc = np.ctypeslib.as_array(lib(b200).igref_cand_scores(h), (n,)).copy() if n else np.zeros(0, np.int64)
        return Candidates(words, sup, sc)
    finally:
        lib(b200).igref_cand_free(h)


def total_score(scores: np.ndarray) -> int:
    scores = np.ascontiguousarray(scores, np.int64)
    out = C.c_int64()
    _check(lib().igref_total_score(_p64(scores), scores.shape[0], C.byref(out)))
    return out.value


@dataclass
class RefRun:
    L: int
    vocab: list
    attack: np.ndarray
    normal: np.ndarray
    tests: np.ndarray | None
    removed_rows: np.ndarray
    cand: list = field(default_factory=list)   # [(words, supports, scores)] attack, normal
    pure: list = field(default_factory=list)
    A: np.ndarray | None = None
    N: np.ndarray | None = None
    labels: np.ndarray | None = None
    regulation: np.ndarray | None = None
    truth: np.ndarray | None = None
    mu: float = 0.0
    sigma: float = 0.0
    times: dict = field(default_factory=dict)
    kind: np.ndarray | None = None
    mean: np.ndarray | None = None
    std: np.ndarray | None = None
    n_train: int = 0
    n_test: int = 0


def run(csv: bytes, label_col: str = "label", attack_values: str = "", normal_values: str = "",
        decimals: int = 1, ratio_k: int = 8, train_rows: int = 0, backend: str = "parallel-cpu",
        threads: int = 0, pair_batch: int = 8192, coverage_block: int = 4096,
        test_limit: int | None = None, stages: int = 2, r: float = 0.568, test_offset: int = 0) -> RefRun:
    """Full reference pipeline: parse → schema → encode → mine → purify → evidence."""
    b200 = backend == "b200"
    L_ = lib(b200)
    h = C.c_void_p()
    tl = (1 << 63) if test_limit is None else test_limit
    _check(L_.igref_run_create(csv, len(csv), label_col.encode(), attack_values.encode(),
                               normal_values.encode(), decimals, ratio_k, train_rows, backend.encode(),
                               threads, pair_batch, coverage_block, test_offset, tl, stages, r, C.byref(h)), b200)
    try:
        L = L_.igref_run_L(h)
        k = (L + 63) // 64

        def mat(which, nrows):
            if nrows == 0:
                return np.zeros((0, k), np.int64)
            return np.ctypeslib.as_array(L_.igref_run_matrix(h, which), (nrows * k,)).reshape(nrows, k).copy()

        na, nn, nt, nrem = (L_.igref_run_rows(h, i) for i in range(4))
        vocab = L_.igref_run_vocab(h).decode().split("\n")[:-1]
        rem = np.ctypeslib.as_array(L_.igref_run_removed(h), (nrem,)).copy() if nrem else np.zeros(0, np.uint64)
        ncols = L_.igref_run_cols(h)
        kind = np.zeros(ncols, np.uint8)
        mean = np.zeros(ncols)
        sd = np.zeros(ncols)
        li = C.c_size_t()
        L_.igref_run_schema(h, kind.ctypes.data_as(C.POINTER(C.c_uint8)),
                            mean.ctypes.data_as(C.POINTER(C.c_double)),
                            sd.ctypes.data_as(C.POINTER(C.c_double)), C.byref(li))
        out = RefRun(L, vocab, mat(0, na), mat(1, nn), mat(2, nt) if stages >= 2 else None, rem,
                     kind=kind, mean=mean, std=sd, n_train=L_.igref_run_rows(h, 4),
                     n_test=L_.igref_run_rows(h, 5))
        t = np.ctypeslib.as_array(L_.igref_run_times(h), (8,)).copy()
        out.times = dict(zip(["parse", "encode", "enumerate", "support", "purify", "match", "test_encode",
                              "total"], t.tolist()))
        if stages >= 1:
            for which, dst in ((0, out.cand), (1, out.cand), (2, out.pure), (3, out.pure)):
                n = L_.igref_run_dict_count(h, which)
                if n == 0:
                    dst.append((np.zeros((0, k), np.int64), np.zeros(0, np.int64), np.zeros(0, np.int64)))
                    continue
                w = np.ctypeslib.as_array(L_.igref_run_dict(h, which, 0), (n * k,)).reshape(n, k).copy()
                s = np.ctypeslib.as_array(L_.igref_run_dict(h, which, 1), (n,)).copy()
                sc = np.ctypeslib.as_array(L_.igref_run_dict(h, which, 2), (n,)).copy()
                dst.append((w, s, sc))
        if stages >= 2 and nt:
            out.A = np.ctypeslib.as_array(L_.igref_run_evidence(h, 0), (nt,)).copy()
            out.N = np.ctypeslib.as_array(L_.igref_run_evidence(h, 1), (nt,)).copy()
            out.labels = np.ctypeslib.as_array(L_.igref_run_labels(h, 0), (nt,)).copy()
            out.regulation = np.ctypeslib.as_array(L_.igref_run_labels(h, 1), (nt,)).copy()
            out.truth = np.ctypeslib.as_array(L_.igref_run_labels(h, 2), (nt,)).copy()
            mu, sg = C.c_double(), C.c_double()
            L_.igref_run_stats(h, C.byref(mu), C.byref(sg))
            out.mu, out.sigma = mu.value, sg.value
        return out
    finally:
        L_.igref_run_free(h)
