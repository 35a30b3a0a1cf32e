"""Synthetic NSL-KDD-shape / CICIDS-shape flow tables (bench + parity workload).

There is no network, so the paper's datasets cannot be fetched; this module
generates the *shape* SURVEY.md §8(d) fixes (the "Inputs" row):

* NSL-shape: 41 feature columns + ``label``.  Columns 1,2,3 categorical
  (3/70/11 values), 19 constant 0, 6,11,13,20,21 binary, 7-10,12,14-18 small
  counts, 22,23 in 0..511, 31,32 in 0..255, 24-30,33-40 rates in {0.00..1.00},
  0,4,5 heavy tailed.  Attack fraction 0.4812 (71,463 / 148,517).
  Rows are drawn by prototype mutation: P prototypes per class, every column
  re-drawn from its marginal with probability m (default P=50, m=0.05).
* CICIDS-shape: 78 numeric columns, attack fraction 0.2 (SURVEY.md A.5 recipe 3
  style: zero-inflated columns drawn from a per-column pool).

Generation is a pure function of (rows, seed, recipe) — the same CSV bytes feed
the CUDA path, the plain-C oracle and the reference (oracle/_ref), which is what
makes their outputs comparable bit for bit.
"""
from __future__ import annotations

import io

import numpy as np

NSL_COLUMNS = [
    "duration", "protocol_type", "service", "flag", "src_bytes", "dst_bytes", "land",
    "wrong_fragment", "urgent", "hot", "num_failed_logins", "logged_in", "num_compromised",
    "root_shell", "su_attempted", "num_root", "num_file_creations", "num_shells",
    "num_access_files", "num_outbound_cmds", "is_host_login", "is_guest_login", "count",
    "srv_count", "serror_rate", "srv_serror_rate", "rerror_rate", "srv_rerror_rate",
    "same_srv_rate", "diff_srv_rate", "srv_diff_host_rate", "dst_host_count",
    "dst_host_srv_count", "dst_host_same_srv_rate", "dst_host_diff_srv_rate",
    "dst_host_same_src_port_rate", "dst_host_srv_diff_host_rate", "dst_host_serror_rate",
    "dst_host_srv_serror_rate", "dst_host_rerror_rate", "dst_host_srv_rerror_rate",
]
assert len(NSL_COLUMNS) == 41

ATTACK_NAMES = ["neptune", "smurf", "satan", "ipsweep", "portsweep", "nmap", "back",
                "teardrop", "warezclient", "pod", "guess_passwd", "buffer_overflow"]
PROTOCOLS = ["tcp", "udp", "icmp"]
SERVICES = [f"svc{i:02d}" for i in range(70)]
FLAGS = ["SF", "S0", "REJ", "RSTR", "RSTO", "SH", "S1", "S2", "RSTOS0", "S3", "OTH"]

_HEAVY = (0, 4, 5)
_BINARY = (6, 11, 13, 20, 21)
_SMALL = (7, 8, 9, 10, 12, 14, 15, 16, 17, 18)
_C511 = (22, 23)
_C255 = (31, 32)
_RATES = tuple(range(24, 31)) + tuple(range(33, 41))


def _nsl_marginal(rng: np.random.Generator, col: int, size: int) -> np.ndarray:
    """Draw `size` raw cell values (as strings) from column `col`'s marginal."""
    if col == 1:
        return np.array(PROTOCOLS, dtype=object)[rng.integers(0, 3, size)]
    if col == 2:
        return np.array(SERVICES, dtype=object)[rng.integers(0, 70, size)]
    if col == 3:
        return np.array(FLAGS, dtype=object)[rng.integers(0, 11, size)]
    if col == 19:
        return np.full(size, "0", dtype=object)
    if col in _BINARY:
        return rng.integers(0, 2, size).astype(str).astype(object)
    if col in _SMALL:
        v = np.where(rng.random(size) < 0.7, 0, rng.geometric(0.35, size))
        return v.astype(str).astype(object)
    if col in _C511:
        return rng.integers(0, 512, size).astype(str).astype(object)
    if col in _C255:
        return rng.integers(0, 256, size).astype(str).astype(object)
    if col in _RATES:
        v = np.where(rng.random(size) < 0.35, np.where(rng.random(size) < 0.5, 0, 100),
                     rng.integers(0, 101, size))
        return np.array([f"{x / 100:.2f}" for x in v], dtype=object)
    if col in _HEAVY:
        zero = rng.random(size) < (0.6 if col == 0 else 0.25)
        v = np.floor(rng.lognormal(4.0 if col == 0 else 6.0, 2.2, size)).astype(np.int64)
        return np.where(zero, 0, v).astype(str).astype(object)
    raise AssertionError(col)


def nsl_table(rows: int, seed: int = 2507, prototypes: int = 50, mutation: float = 0.05,
              attack_fraction: float = 0.4812) -> tuple[list[str], np.ndarray]:
    """Return (header, cells[rows, 42] of str) for an NSL-shape table."""
    rng = np.random.default_rng(seed)
    ncol = 41
    protos = np.empty((2, prototypes, ncol), dtype=object)
    for c in range(2):
        for j in range(ncol):
            protos[c, :, j] = _nsl_marginal(rng, j, prototypes)
    proto_label = np.array(ATTACK_NAMES, dtype=object)[rng.integers(0, len(ATTACK_NAMES), prototypes)]
    attack = rng.random(rows) < attack_fraction
    pid = rng.integers(0, prototypes, rows)
    cls = np.where(attack, 0, 1)
    cells = protos[cls, pid, :].copy()
    mutate = rng.random((rows, ncol)) < mutation
    for j in range(ncol):
        idx = np.nonzero(mutate[:, j])[0]
        if idx.size:
            cells[idx, j] = _nsl_marginal(rng, j, idx.size)
    labels = np.where(attack, proto_label[pid], "normal").astype(object)
    out = np.concatenate([cells, labels[:, None]], axis=1)
    return NSL_COLUMNS + ["label"], out


def cicids_table(rows: int, seed: int = 2507, prototypes: int = 1000, mutation: float = 0.01,
                 pool: int = 4000, attack_fraction: float = 0.2) -> tuple[list[str], np.ndarray]:
    """CICIDS-shape: 78 numeric columns, zero-inflated, per-column value pool."""
    rng = np.random.default_rng(seed)
    ncol = 78
    pools = []
    for j in range(ncol):
        if j % 5 == 4:
            pools.append(np.array(["0"] * 19 + ["1"], dtype=object))
        elif j in (7, 33, 61):
            pools.append(np.array(["0"], dtype=object))
        elif j == 0:
            pools.append(np.array(["80", "443", "53", "22", "21", "8080", "123"], dtype=object))
        else:
            vals = np.round(np.where(rng.random(pool) < 0.4, 0.0, rng.lognormal(3.0, 2.5, pool)), 1)
            pools.append(np.array([f"{v:.1f}" for v in vals], dtype=object))

    def draw(j, size):
        return pools[j][rng.integers(0, len(pools[j]), size)]

    protos = np.empty((2, prototypes, ncol), dtype=object)
    for c in range(2):
        for j in range(ncol):
            protos[c, :, j] = draw(j, prototypes)
    attack = rng.random(rows) < attack_fraction
    pid = rng.integers(0, prototypes, rows)
    cells = protos[np.where(attack, 0, 1), pid, :].copy()
    mutate = rng.random((rows, ncol)) < mutation
    for j in range(ncol):
        idx = np.nonzero(mutate[:, j])[0]
        if idx.size:
            cells[idx, j] = draw(j, idx.size)
    labels = np.where(attack, "attack", "BENIGN").astype(object)
    header = [f"f{j}" for j in range(ncol)] + ["Label"]
    return header, np.concatenate([cells, labels[:, None]], axis=1)


def to_csv_bytes(header: list[str], cells: np.ndarray) -> bytes:
    """Plain RFC-4180 CSV (no quoting needed for generated values), LF records."""
    buf = io.StringIO()
    buf.write(",".join(header))
    buf.write("\n")
    for row in cells:
        buf.write(",".join(row))
        buf.write("\n")
    return buf.getvalue().encode()


def nsl_csv(rows: int, seed: int = 2507, **kw) -> bytes:
    return to_csv_bytes(*nsl_table(rows, seed, **kw))


def cicids_csv(rows: int, seed: int = 2507, **kw) -> bytes:
    return to_csv_bytes(*cicids_table(rows, seed, **kw))
