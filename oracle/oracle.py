"""ctypes driver for the plain-C oracle (oracle/ig_oracle.c) — TEST INFRASTRUCTURE ONLY.

The checker the CUDA path is compared with.  Only tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline leg may import it.  `fit()` composes the restated
mine → score → purify sequence exactly as the reference's
CLI `cmd_train` would.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "_build", "libigoracle.so")

_lib = None


class OracleError(RuntimeError):
    def __init__(self, status):
        super().__init__(f"oracle status {status}")
        self.status = status


def build() -> str:
    subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)
    return SO


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(SO):
            build()
        L = C.CDLL(SO)
        p64 = C.POINTER(C.c_int64)
        sz = C.c_size_t
        L.igo_enumerate.argtypes = [p64, sz, sz, C.c_int, C.POINTER(C.c_void_p)]
        L.igo_set_count.argtypes = [C.c_void_p]
        L.igo_set_count.restype = sz
        L.igo_set_words.argtypes = [C.c_void_p]
        L.igo_set_words.restype = p64
        L.igo_set_free.argtypes = [C.c_void_p]
        L.igo_count_support.argtypes = [p64, sz, p64, sz, sz, C.c_int, p64]
        L.igo_score.argtypes = [p64, p64, sz, sz, p64]
        L.igo_total_score.argtypes = [p64, sz, p64]
        L.igo_coverage_any.argtypes = [p64, sz, p64, sz, sz, C.c_int, C.POINTER(C.c_uint8)]
        L.igo_fused_score.argtypes = [p64, p64, sz, p64, sz, sz, C.c_int, p64]
        L.igo_reject_covered.argtypes = [p64, p64, p64, sz, p64, sz, sz, C.c_int]
        L.igo_reject_covered.restype = sz
        _lib = L
    return _lib


def _w(a):
    a = np.ascontiguousarray(a, dtype=np.int64)
    if a.ndim == 1:
        a = a.reshape(0, 1) if a.size == 0 else a.reshape(1, -1)
    return a


def _p(a):
    return a.ctypes.data_as(C.POINTER(C.c_int64))


def _chk(st):
    if st:
        raise OracleError(st)


def enumerate_candidates(rows: np.ndarray, threads: int = 0) -> np.ndarray:
    rows = _w(rows)
    k = rows.shape[1]
    h = C.c_void_p()
    _chk(lib().igo_enumerate(_p(rows), rows.shape[0], k, threads, C.byref(h)))
    try:
        n = lib().igo_set_count(h)
        if n == 0:
            return np.zeros((0, k), np.int64)
        return np.ctypeslib.as_array(lib().igo_set_words(h), (n * k,)).reshape(n, k).copy()
    finally:
        lib().igo_set_free(h)


def count_support(pat, rows, threads: int = 0) -> np.ndarray:
    pat, rows = _w(pat), _w(rows)
    out = np.zeros(pat.shape[0], np.int64)
    _chk(lib().igo_count_support(_p(pat), pat.shape[0], _p(rows), rows.shape[0], pat.shape[1], threads, _p(out)))
    return out


def score_patterns(pat, support) -> np.ndarray:
    pat = _w(pat)
    support = np.ascontiguousarray(support, np.int64)
    out = np.zeros(pat.shape[0], np.int64)
    _chk(lib().igo_score(_p(pat), _p(support), pat.shape[0], pat.shape[1], _p(out)))
    return out


def total_score(s) -> int:
    s = np.ascontiguousarray(s, np.int64)
    out = C.c_int64()
    _chk(lib().igo_total_score(_p(s), s.shape[0], C.byref(out)))
    return out.value


def coverage_any(pat, opp, threads: int = 0) -> np.ndarray:
    pat, opp = _w(pat), _w(opp)
    mask = np.zeros(pat.shape[0], np.uint8)
    _chk(lib().igo_coverage_any(_p(pat), pat.shape[0], _p(opp), opp.shape[0], pat.shape[1], threads,
                                mask.ctypes.data_as(C.POINTER(C.c_uint8))))
    return mask


def fused_score(pat, scores, tests, threads: int = 0) -> np.ndarray:
    pat, tests = _w(pat), _w(tests)
    scores = np.ascontiguousarray(scores, np.int64)
    out = np.zeros(tests.shape[0], np.int64)
    _chk(lib().igo_fused_score(_p(pat), _p(scores), pat.shape[0], _p(tests), tests.shape[0], pat.shape[1],
                               threads, _p(out)))
    return out


@dataclass
class Dictionary:
    words: np.ndarray
    supports: np.ndarray
    scores: np.ndarray


@dataclass
class Fit:
    candidates: list  # [Dictionary attack, Dictionary normal]
    pure: list


def fit(attack: np.ndarray, normal: np.ndarray, threads: int = 0) -> Fit:
    """cmd_train's mining half: mine both classes, purify both ways."""
    X = [_w(attack), _w(normal)]
    cands, pures = [], []
    for c in range(2):
        w = enumerate_candidates(X[c], threads)
        s = count_support(w, X[c], threads)
        sc = score_patterns(w, s)
        total_score(sc)
        cands.append(Dictionary(w, s, sc))
    for c in range(2):
        d = cands[c]
        keep = coverage_any(d.words, X[1 - c], threads) == 0
        pures.append(Dictionary(d.words[keep], d.supports[keep], d.scores[keep]))
    return Fit(cands, pures)
