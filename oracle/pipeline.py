"""Pure-Python restatement of the reference dataset pipeline — TEST INFRASTRUCTURE ONLY.

Restates, for small inputs, the tokenise → vocabulary → filter → pack path of
the reference so the CUDA tokeniser (kernel 1) can be checked without the
reference present:

  read_csv               proj/src/csv.cpp:14-89     (RFC 4180, BOM strip, ragged → DataError)
  parse_double_strict    proj/src/pipeline.cpp:16-25 (std::from_chars, whole cell, finite)
  format_zscore          proj/src/pipeline.cpp:77-105
  infer_schema           proj/src/pipeline.cpp:107-169 (sequential sums, population std)
  tokenize_row           proj/src/pipeline.cpp:171-202
  TokenVocabulary.build  proj/src/pipeline.cpp:62-69 (std::set byte order)
  anti_contradiction     proj/src/pipeline.cpp:204-235
  encode_training        proj/src/pipeline.cpp:273-328 (vocab built BEFORE filtering)
  encode_rows            proj/src/pipeline.cpp:330-339 (unseen tokens dropped)
  is_attack              proj/src/pipeline.cpp:35-49

Pinned against oracle/_ref (the reference compiled) by tests/golden/make_golden.py.
Plus the spec-only infer/eval arithmetic.
"""
from __future__ import annotations

import ctypes
import ctypes.util
import math
import re
from dataclasses import dataclass, field

import numpy as np

# Correctly rounded fused multiply-add (C99 fma from libm; Python 3.12 has no
# math.fma).  The reference is compiled with -march=native
# (proj/CMakeLists.txt:10-18): GCC contracts `ss += d * d` (pipeline.cpp:159)
# into vfmadd231sd, so the standard deviation rounds once per term.
_libm = ctypes.CDLL(ctypes.util.find_library("m") or "libm.so.6")
_libm.fma.restype = ctypes.c_double
_libm.fma.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_double]
fma = _libm.fma


class DataError(Exception):
    pass


class ConfigError(Exception):
    pass


# ---------------------------------------------------------------- csv.cpp:14-89
def read_csv(text: bytes, origin: str = "<stream>"):
    if text[:3] == b"\xef\xbb\xbf":
        text = text[3:]
    s = text.decode("utf-8", errors="surrogateescape")
    header = None
    rows = []
    record, fld = [], []
    in_q = False
    any_field = False
    line = 1
    i, n = 0, len(s)

    def end_record():
        nonlocal header, record, any_field
        record.append("".join(fld))
        fld.clear()
        if header is None:
            header = record
        else:
            if len(record) != len(header):
                raise DataError(f"{origin}: line {line}: expected {len(header)} fields, got {len(record)}")
            rows.append(record)
        record = []
        any_field = False

    while i < n:
        c = s[i]
        if in_q:
            if c == '"':
                if i + 1 < n and s[i + 1] == '"':
                    fld.append('"')
                    i += 1
                else:
                    in_q = False
            else:
                if c == "\n":
                    line += 1
                fld.append(c)
            i += 1
            continue
        if c == '"':
            in_q = True
        elif c == ",":
            record.append("".join(fld))
            fld.clear()
            any_field = True
        elif c == "\r" or c == "\n":
            if c == "\r" and i + 1 < n and s[i + 1] == "\n":
                i += 1
            end_record()
            line += 1
        else:
            fld.append(c)
        i += 1
    if in_q:
        raise DataError(f"{origin}: unterminated quoted field at end of input")
    if any_field or fld:
        end_record()
    if header is None:
        raise DataError(f"{origin}: empty input, no header row")
    return header, rows


# ---------------------------------------------------------------- pipeline.cpp:16-25
_NUM = re.compile(r"-?(?:\d+\.?\d*|\.\d+)(?:[eE][+-]?\d+)?\Z")


def parse_double_strict(cell: str):
    if not cell or not _NUM.match(cell):
        return None
    v = float(cell)
    if not math.isfinite(v):
        return None
    return v


# ---------------------------------------------------------------- pipeline.cpp:77-105
def zscore_units(z: float, decimals: int) -> int:
    scaled = z * (10.0 ** decimals)
    cap = 9.0e18
    if abs(scaled) >= cap:
        return -int(cap) if scaled < 0 else int(cap)
    t = math.trunc(scaled)
    if abs(scaled - t) >= 0.5:  # llround: halfway away from zero
        t += 1 if scaled > 0 else -1
    return int(t)


def format_units(units: int, decimals: int) -> str:
    denom = 10 ** decimals
    neg = units < 0
    mag = -units if neg else units
    whole, frac = divmod(mag, denom)
    out = "-" if (neg and mag != 0) else ""
    out += str(whole)
    if decimals > 0:
        out += "." + str(frac).rjust(decimals, "0")
    return out


def format_zscore(z: float, decimals: int) -> str:
    return format_units(zscore_units(z, decimals), decimals)


# ---------------------------------------------------------------- pipeline.cpp:35-49,107-169
@dataclass
class Schema:
    names: list
    kind: list  # "numeric" | "categorical"
    mean: list
    std: list
    label_index: int
    attack_values: list = field(default_factory=list)
    normal_values: list = field(default_factory=list)
    decimals: int = 2

    def is_attack(self, label: str) -> bool:
        if self.attack_values:
            if label in self.attack_values:
                return True
            if not self.normal_values or label in self.normal_values:
                return False
            raise DataError(f"label value '{label}' not covered by attack/normal mapping")
        if self.normal_values:
            return label not in self.normal_values
        return label != "normal"


def infer_schema(header, rows, label_column, attack_values=(), normal_values=(), decimals=2) -> Schema:
    if not rows:
        raise DataError("empty table: no data rows to train on")
    if decimals < 0 or decimals > 12:
        raise ConfigError(f"decimals must be in [0, 12], got {decimals}")
    if label_column not in header:
        raise ConfigError(f"label column '{label_column}' not found in header")
    li = header.index(label_column)
    kind, mean, std = [], [], []
    for j in range(len(header)):
        if j == li:
            kind.append("categorical"), mean.append(0.0), std.append(0.0)
            continue
        numeric, parsed, s = True, 0, 0.0
        for r in rows:
            cell = r[j]
            if not cell:
                continue
            v = parse_double_strict(cell)
            if v is None:
                numeric = False
                break
            s += v
            parsed += 1
        if not numeric or parsed == 0:
            kind.append("categorical"), mean.append(0.0), std.append(0.0)
            continue
        m = s / parsed
        ss = 0.0
        for r in rows:
            cell = r[j]
            if not cell:
                continue
            d = parse_double_strict(cell) - m
            ss = fma(d, d, ss)  # the reference's -march=native build contracts pipeline.cpp:159
        kind.append("numeric"), mean.append(m), std.append(math.sqrt(ss / parsed))
    sch = Schema(list(header), kind, mean, std, li, list(attack_values), list(normal_values), decimals)
    for r in rows:
        sch.is_attack(r[li])
    return sch


# ---------------------------------------------------------------- pipeline.cpp:171-202
def tokenize_row(row, schema: Schema, row_index=0):
    if len(row) != len(schema.names):
        raise DataError(f"row {row_index}: expected {len(schema.names)} columns, got {len(row)}")
    toks = []
    for j, cell in enumerate(row):
        if j == schema.label_index:
            continue
        if not cell:
            value = ""
        elif schema.kind[j] == "numeric":
            v = parse_double_strict(cell)
            if v is None:
                raise DataError(f"row {row_index}, column {j} ({schema.names[j]}): cannot parse '{cell}' as a number")
            z = 0.0 if schema.std[j] == 0.0 else (v - schema.mean[j]) / schema.std[j]
            value = format_zscore(z, schema.decimals)
        else:
            value = cell
        toks.append(f"{j}:{value}")
    return toks


def _sortkey(tok: str) -> bytes:
    return tok.encode("utf-8", errors="surrogateescape")


def pack(bits, L: int) -> np.ndarray:
    k = (L + 63) // 64
    w = np.zeros(k, np.uint64)
    for b in bits:
        if b >= L:
            raise IndexError(f"bit index {b} out of range for logical length {L}")
        w[b // 64] |= np.uint64(1) << np.uint64(b % 64)
    return w.view(np.int64)


@dataclass
class TrainingEncoding:
    vocab: list
    attack: np.ndarray
    normal: np.ndarray
    removed_rows: list
    L: int


def encode_training(rows, schema: Schema) -> TrainingEncoding:
    token_sets = [tokenize_row(r, schema, i) for i, r in enumerate(rows)]
    vocab = sorted({t for ts in token_sets for t in ts}, key=_sortkey)
    index = {t: i for i, t in enumerate(vocab)}
    inst = []
    for i, (r, ts) in enumerate(zip(rows, token_sets)):
        inst.append((tuple(sorted(index[t] for t in ts)), schema.is_attack(r[schema.label_index]), i))
    if not any(a for _, a, _ in inst) or all(a for _, a, _ in inst):
        raise DataError("training data must contain both attack and normal instances")
    by_sig = {}
    for bits, a, _ in inst:
        c = by_sig.setdefault(bits, [0, 0])
        c[0 if a else 1] += 1
    bad = {b for b, c in by_sig.items() if c[0] > 0 and c[1] > 0}
    removed = sorted(i for bits, _, i in inst if bits in bad)
    kept = [x for x in inst if x[0] not in bad]
    if not any(a for _, a, _ in kept) or all(a for _, a, _ in kept):
        raise DataError("anti-contradiction filtering emptied a class; training impossible")
    L = len(vocab)
    k = (L + 63) // 64
    att = [pack(b, L) for b, a, _ in kept if a]
    nor = [pack(b, L) for b, a, _ in kept if not a]
    att = np.stack(att) if att else np.zeros((0, k), np.int64)
    nor = np.stack(nor) if nor else np.zeros((0, k), np.int64)
    return TrainingEncoding(vocab, att, nor, removed, L)


def encode_rows(rows, schema: Schema, vocab) -> np.ndarray:
    index = {t: i for i, t in enumerate(vocab)}
    L = len(vocab)
    k = (L + 63) // 64
    out = np.zeros((len(rows), k), np.int64)
    for i, r in enumerate(rows):
        out[i] = pack(sorted(index[t] for t in tokenize_row(r, schema, i) if t in index), L)
    return out


def truth_labels(rows, schema: Schema) -> np.ndarray:
    return np.array([1 if schema.is_attack(r[schema.label_index]) else 0 for r in rows], np.uint8)


# ---------------------------------------------------------------- SPEC.md:434-452 (infer)
def fit_normal_stats(nvals) -> tuple[float, float]:
    pos = [float(v) for v in nvals if v > 0]
    if len(pos) < 2:
        return 0.0, 0.0
    s = 0.0
    for v in pos:
        s += v
    mu = s / len(pos)
    ss = 0.0
    for v in pos:
        ss = fma(v - mu, v - mu, ss)  # as the FMA-contracted restatement in oracle/ref_shim.cpp
    return mu, math.sqrt(ss / len(pos))


def classify(a: int, n: int, mu: float, sigma: float, r: float) -> tuple[int, int]:
    """(label, regulation): 1=R1-attack 2=R1-normal 3=R2 4=R3."""
    if a == 0 and n == 0:
        return 1, 3
    if a >= n:
        return 1, 1
    if float(n) < fma(-r, sigma, mu):  # mu - r*sigma, contracted like oracle/ref_shim.cpp's build
        return 1, 4
    return 0, 2


# ---------------------------------------------------------------- SPEC.md:518-526 (eval)
def compute_metrics(pred, truth, margins) -> dict:
    pred = np.asarray(pred).astype(bool)
    truth = np.asarray(truth).astype(bool)
    tp = int(np.sum(pred & truth))
    fp = int(np.sum(pred & ~truth))
    tn = int(np.sum(~pred & ~truth))
    fn = int(np.sum(~pred & truth))
    tot = tp + fp + tn + fn
    acc = (tp + tn) / tot if tot else 0.0
    rec = tp / (tp + fn) if tp + fn else 0.0
    prec = tp / (tp + fp) if tp + fp else 0.0
    f1 = 2 * prec * rec / (prec + rec) if prec + rec else 0.0
    tpr = rec
    tnr = tn / (tn + fp) if tn + fp else 0.0
    m = np.asarray(margins, dtype=np.float64)
    pos, neg = m[truth], m[~truth]
    if len(pos) and len(neg):
        order = np.sort(neg)
        less = np.searchsorted(order, pos, side="left")
        leq = np.searchsorted(order, pos, side="right")
        auc = float((less.sum() + 0.5 * (leq - less).sum()) / (len(pos) * len(neg)))
    else:
        auc = 0.0
    return dict(tp=tp, fp=fp, tn=tn, fn=fn, accuracy=acc, recall=rec, precision=prec, f1=f1,
                balanced_auc=(tpr + tnr) / 2, rank_auc=auc)
