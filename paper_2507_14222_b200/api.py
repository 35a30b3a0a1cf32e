"""Python mirror of the reference interface for the IG hot path, over the C-ABI.

Names, argument meaning and error behaviour follow the reference:

* ``KernelBackend`` / ``make_backend`` / ``backend_names`` — proj/include/ig/kernels.hpp:27-58
* ``KernelConfig`` — kernels.hpp:14-21 (validated like kernels.cpp:12-15)
* ``enumerate_candidates`` / ``count_support`` / ``score_patterns`` / ``total_score``
  — proj/include/ig/mine.hpp:35-51
* ``read_csv`` / ``infer_schema`` / ``encode_training`` / ``encode_rows`` — csv.hpp:19,
  pipeline.hpp:70-109
* ``reject_covered``, ``evidence_scores``,
  ``fit_normal_stats`` / ``classify``, ``compute_metrics``

Exceptions: std::invalid_argument → ValueError, std::out_of_range → IndexError,
ig::ConfigError → ConfigError, ig::DataError → DataError, ig::ArithmeticError →
IGArithmeticError (a builtin ArithmeticError), CUDA failures → CudaError.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from . import _native as N

lib = N.lib


class ConfigError(Exception):
    pass


class IoError(OSError):
    pass


class DataError(Exception):
    pass


class IGArithmeticError(ArithmeticError):
    pass


class CudaError(RuntimeError):
    pass


_STATUS = {1: ValueError, 2: IndexError, 3: ConfigError, 4: IoError, 5: DataError, 6: IGArithmeticError,
           7: CudaError, 8: CudaError, 9: MemoryError}


def _raise(status: int, ctx=None):
    msg = lib.ig_last_error(ctx.handle if ctx is not None else None)
    msg = msg.decode() if msg else ""
    raise _STATUS.get(status, CudaError)(msg)


def _p64(a: np.ndarray):
    return a.ctypes.data_as(N.p64)


def _words(a, L: int) -> np.ndarray:
    k = (L + 63) // 64
    a = np.ascontiguousarray(a, dtype=np.int64)
    if a.size == 0:
        return np.zeros((0, k), np.int64)
    return a.reshape(-1, k)


@dataclass
class KernelConfig:
    """kernels.hpp:14-21.  Batch sizes never change results."""
    pair_batch: int = 8192
    coverage_block: int = 4096
    memory_budget_bytes: int = 2 << 30
    threads: int = 0

    def validate(self):
        if self.pair_batch < 1:
            raise ConfigError("pair-batch must be >= 1")
        if self.coverage_block < 1:
            raise ConfigError("coverage-block must be >= 1")

    def c(self):
        self.validate()
        return N.KernelConfigC(self.pair_batch, self.coverage_block, self.memory_budget_bytes, self.threads)


class Context:
    """One device + stream.  All calls of one Context run in order on its stream."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        st = lib.ig_ctx_create(device, C.byref(h))
        if st:
            _raise(st)
        self.handle = h
        self.device = device
        self.stream = None  # None = the context's own stream

    def set_stream(self, stream) -> None:
        ptr = getattr(stream, "cuda_stream", stream)
        st = lib.ig_ctx_set_stream(self.handle, C.c_void_p(ptr or None))
        if st:
            _raise(st, self)
        self.stream = ptr or None

    def on_stream(self, stream):
        """Context manager: run this context's work on `stream` (e.g. torch's
        current stream, so that buffers torch produced are ordered before the
        library reads them), restoring the previous stream afterwards."""
        import contextlib

        @contextlib.contextmanager
        def cm():
            prev = self.stream
            self.set_stream(stream)
            try:
                yield self
            finally:
                self.set_stream(prev)
        return cm()

    @property
    def launches(self) -> int:
        return int(lib.ig_ctx_launch_count(self.handle))

    def set_diagnostics(self, on: bool) -> None:
        self.check(lib.ig_ctx_set_diagnostics(self.handle, 1 if on else 0))

    DIAG_KERNELS = ("pair_enum", "support", "cover", "match")

    def diag_kernel(self, kernel: str) -> tuple[float, int, int]:
        """(kernel ms, exact useful 64-bit word-ANDs, launches) of one hot kernel
        ("pair_enum", "support", "cover", "match") since set_diagnostics(True)."""
        ms, w, n = C.c_double(), C.c_uint64(), C.c_uint64()
        self.check(lib.ig_ctx_diag_kernel(self.handle, self.DIAG_KERNELS.index(kernel), C.byref(ms), C.byref(w),
                                          C.byref(n)))
        return ms.value, int(w.value), int(n.value)

    def int_peaks(self) -> tuple[float, float]:
        """Measured (LOP3.32/s, POPC.32/s) of this device (diag.cu)."""
        a, b = C.c_double(), C.c_double()
        self.check(lib.ig_measure_int_peaks(self.handle, C.byref(a), C.byref(b)))
        return a.value, b.value

    def check(self, status: int):
        if status:
            _raise(status, self)

    def close(self):
        if self.handle:
            lib.ig_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ctx: Optional[Context] = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


@dataclass
class PackedMatrix:
    """Class-contiguous n x K int64 rows (bitpack.hpp:114-141)."""
    words: np.ndarray
    logical_len: int
    class_tag: str = "unlabeled"

    def __post_init__(self):
        self.words = _words(self.words, self.logical_len)

    @property
    def rows(self) -> int:
        return self.words.shape[0]

    @property
    def word_count(self) -> int:
        return (self.logical_len + 63) // 64


def _mat(x, L=None) -> PackedMatrix:
    if isinstance(x, PackedMatrix):
        return x
    if L is None:
        raise ValueError("logical_len required for raw arrays")
    return PackedMatrix(x, L)


class KernelBackend:
    """The 'b200' KernelBackend (kernels.hpp:27-53) over the C-ABI."""

    def __init__(self, ctx: Optional[Context] = None):
        self.ctx = ctx or default_context()

    def name(self) -> str:
        return "b200"

    def pair_intersect_batch(self, rows: PackedMatrix, left: int, j_begin: int, j_end: int) -> np.ndarray:
        out = np.zeros((max(j_end - j_begin, 0), rows.word_count), np.int64)
        self.ctx.check(lib.ig_pair_intersect_batch(self.ctx.handle, _p64(rows.words), rows.rows, rows.logical_len,
                                                   left, j_begin, j_end, _p64(out)))
        return out

    def coverage_any(self, patterns: PackedMatrix, opponents: PackedMatrix, coverage_block: int = 4096) -> np.ndarray:
        mask = np.zeros(patterns.rows, np.uint8)
        self.ctx.check(lib.ig_coverage_any(self.ctx.handle, _p64(patterns.words), patterns.rows,
                                           patterns.logical_len, _p64(opponents.words), opponents.rows,
                                           opponents.logical_len, coverage_block, mask.ctypes.data_as(N.pu8)))
        return mask

    def fused_score(self, patterns: PackedMatrix, scores, tests: PackedMatrix) -> np.ndarray:
        scores = np.ascontiguousarray(scores, np.int64)
        out = np.zeros(tests.rows, np.int64)
        self.ctx.check(lib.ig_fused_score(self.ctx.handle, _p64(patterns.words), patterns.rows, patterns.logical_len,
                                          _p64(scores), scores.shape[0], _p64(tests.words), tests.rows,
                                          tests.logical_len, _p64(out)))
        return out


def backend_names() -> list[str]:
    return ["b200"]


def make_backend(name: str, threads: int = 0, ctx: Optional[Context] = None) -> KernelBackend:
    """kernels.hpp:55-57: unknown names raise ConfigError listing the available ones."""
    if name == "b200":
        return KernelBackend(ctx)
    raise ConfigError(f"unknown backend '{name}'; available: " + " ".join(backend_names()))


@dataclass
class CandidateSet:
    """mine.hpp:21-29: deduplicated candidates of one class in canonical bit order."""
    class_tag: str
    patterns: PackedMatrix
    supports: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))
    scores: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))
    source_rows: int = 0
    _handle: object = None
    _ctx: object = None

    def __del__(self):
        if self._handle and lib is not None:
            lib.ig_candidates_free(self._handle)
            self._handle = None


def enumerate_candidates(rows: PackedMatrix, backend: Optional[KernelBackend] = None,
                         config: Optional[KernelConfig] = None,
                         progress: Optional[Callable[[int, int, int], None]] = None) -> CandidateSet:
    backend = backend or KernelBackend()
    config = config or KernelConfig()
    ctx = backend.ctx
    cfg = config.c()
    h = C.c_void_p()
    cb = N.PROGRESS((lambda d, t, f, u: progress(d, t, f)) if progress else (lambda d, t, f, u: None))
    ctx.check(lib.ig_enumerate_candidates(ctx.handle, _p64(rows.words), rows.rows, rows.logical_len, C.byref(cfg),
                                          cb, None, C.byref(h)))
    n = lib.ig_candidates_count(h)
    words = np.zeros((n, rows.word_count), np.int64)
    ctx.check(lib.ig_candidates_copy(ctx.handle, h, _p64(words), None, None))
    return CandidateSet(rows.class_tag, PackedMatrix(words, rows.logical_len, rows.class_tag),
                        source_rows=rows.rows, _handle=h, _ctx=ctx)


def count_support(candidates: CandidateSet, rows: PackedMatrix, config: Optional[KernelConfig] = None) -> None:
    config = config or KernelConfig()
    ctx = candidates._ctx
    cfg = config.c()
    ctx.check(lib.ig_count_support(ctx.handle, candidates._handle, _p64(rows.words), rows.rows, rows.logical_len,
                                   C.byref(cfg)))
    sup = np.zeros(candidates.patterns.rows, np.int64)
    ctx.check(lib.ig_candidates_copy(ctx.handle, candidates._handle, None, _p64(sup), None))
    candidates.supports = sup


def score_patterns(candidates: CandidateSet) -> None:
    ctx = candidates._ctx
    ctx.check(lib.ig_score_patterns(ctx.handle, candidates._handle))
    sc = np.zeros(candidates.patterns.rows, np.int64)
    ctx.check(lib.ig_candidates_copy(ctx.handle, candidates._handle, None, None, _p64(sc)))
    candidates.scores = sc


def total_score(scores) -> int:
    s = np.ascontiguousarray(scores, np.int64)
    out = C.c_int64()
    st = lib.ig_total_score(_p64(s), s.shape[0], C.byref(out))
    if st:
        _raise(st)
    return out.value


# ---------------------------------------------------------------- fit / evidence
@dataclass
class Dictionary:
    words: np.ndarray
    supports: np.ndarray
    scores: np.ndarray


class _PinnedBlock:
    """One page-locked block of the library's host pool (ig_host_alloc)."""
    __slots__ = ("ptr",)

    def __init__(self, nbytes: int):
        p = C.c_void_p()
        st = lib.ig_host_alloc(nbytes, C.byref(p))
        if st:
            _raise(st, None)
        self.ptr = p.value

    def __del__(self):
        if self.ptr and lib is not None:  # lib is None at interpreter teardown
            lib.ig_host_free(C.c_void_p(self.ptr))
            self.ptr = None


def pinned_array(shape, dtype) -> np.ndarray:
    """numpy array in page-locked host memory; the block returns to the pool
    when the last view of it is gone."""
    dtype = np.dtype(dtype)
    nbytes = int(np.prod(shape)) * dtype.itemsize
    if nbytes == 0:
        return np.zeros(shape, dtype)
    blk = _PinnedBlock(nbytes)
    buf = (C.c_char * nbytes).from_address(blk.ptr)
    buf._ig_block = blk  # the array's base keeps the block alive
    return np.frombuffer(buf, dtype=dtype, count=int(np.prod(shape))).reshape(shape)


class Model:
    """Pure dictionaries P+ / P- (and candidate sets B+ / B-) resident on the device."""

    def __init__(self, ctx: Context, handle):
        self.ctx = ctx
        self.handle = handle
        self.logical_len = int(lib.ig_model_logical_len(handle))

    def count(self, cls: int, which: int) -> int:
        return int(lib.ig_model_count(self.handle, cls, which))

    def dictionary(self, cls: int, which: int = 1) -> Dictionary:
        """cls 0 attack / 1 normal; which 0 candidates B^c / 1 pure P^c.  The
        arrays live in page-locked host memory (reused across calls once freed)."""
        n = self.count(cls, which)
        k = (self.logical_len + 63) // 64
        w = pinned_array((n, k), np.int64)
        s = pinned_array((n,), np.int64)
        sc = pinned_array((n,), np.int64)
        self.ctx.check(lib.ig_model_copy(self.ctx.handle, self.handle, cls, which, _p64(w), _p64(s), _p64(sc)))
        return Dictionary(w, s, sc)

    def phase_ms(self) -> dict:
        a = (C.c_double * 6)()
        lib.ig_model_phase_ms(self.handle, a)
        return dict(zip(["rows", "enumerate", "support", "purify", "order", "total"], list(a)))

    def evidence(self, tests) -> tuple[np.ndarray, np.ndarray]:
        """evidence_scores on host rows."""
        t = _mat(tests, self.logical_len)
        A = np.zeros(t.rows, np.int64)
        Nn = np.zeros(t.rows, np.int64)
        self.ctx.check(lib.ig_evidence(self.ctx.handle, self.handle, _p64(t.words), t.rows, t.logical_len,
                                       _p64(A), _p64(Nn)))
        return A, Nn

    def evidence_device(self, d_tests_ptr: int, n_tests: int, d_A_ptr: int, d_N_ptr: int) -> None:
        self.ctx.check(lib.ig_evidence_device(self.ctx.handle, self.handle, C.c_void_p(d_tests_ptr), n_tests,
                                              self.logical_len, C.c_void_p(d_A_ptr), C.c_void_p(d_N_ptr)))

    def evidence_encoded_device(self, enc: "Encoding", d_A_ptr: int, d_N_ptr: int) -> None:
        """evidence of a test encoding into device int64 buffers (ordered on the context stream)."""
        self.ctx.check(lib.ig_evidence_encoded_device(self.ctx.handle, self.handle, enc.handle,
                                                      C.c_void_p(d_A_ptr), C.c_void_p(d_N_ptr)))

    def evidence_encoded(self, enc: "Encoding") -> tuple[np.ndarray, np.ndarray]:
        n = enc.rows(2)
        A = pinned_array((n,), np.int64)
        Nn = pinned_array((n,), np.int64)
        self.ctx.check(lib.ig_evidence_encoded(self.ctx.handle, self.handle, enc.handle, _p64(A), _p64(Nn)))
        return A, Nn

    def __del__(self):
        if getattr(self, "handle", None) and lib is not None:  # lib is None at interpreter teardown
            lib.ig_model_free(self.handle)
            self.handle = None


def fit(attack, normal, logical_len: int, config: Optional[KernelConfig] = None,
        ctx: Optional[Context] = None) -> Model:
    ctx = ctx or default_context()
    cfg = (config or KernelConfig()).c()
    a, n = _words(attack, logical_len), _words(normal, logical_len)
    h = C.c_void_p()
    ctx.check(lib.ig_fit(ctx.handle, _p64(a), a.shape[0], _p64(n), n.shape[0], logical_len, C.byref(cfg),
                         C.byref(h)))
    return Model(ctx, h)


def fit_device(d_attack_ptr: int, n_attack: int, d_normal_ptr: int, n_normal: int, logical_len: int,
               config: Optional[KernelConfig] = None, ctx: Optional[Context] = None) -> Model:
    ctx = ctx or default_context()
    cfg = (config or KernelConfig()).c()
    h = C.c_void_p()
    ctx.check(lib.ig_fit_device(ctx.handle, C.c_void_p(d_attack_ptr), n_attack, C.c_void_p(d_normal_ptr), n_normal,
                                logical_len, C.byref(cfg), C.byref(h)))
    return Model(ctx, h)


def reject_covered(candidates: CandidateSet, opposite: PackedMatrix, backend: Optional[KernelBackend] = None,
                   coverage_block: int = 4096) -> CandidateSet:
    """keep the candidates coverage_any reports not covered."""
    backend = backend or KernelBackend()
    keep = backend.coverage_any(candidates.patterns, opposite, coverage_block) == 0
    return CandidateSet(candidates.class_tag,
                        PackedMatrix(candidates.patterns.words[keep], candidates.patterns.logical_len,
                                     candidates.class_tag),
                        candidates.supports[keep] if candidates.supports.size else candidates.supports,
                        candidates.scores[keep] if candidates.scores.size else candidates.scores,
                        candidates.source_rows)


# ---------------------------------------------------------------- pipeline (kernel 1)
class Table:
    def __init__(self, handle):
        self.handle = handle

    @property
    def rows(self) -> int:
        return int(lib.ig_table_rows(self.handle))

    @property
    def columns(self) -> int:
        return int(lib.ig_table_cols(self.handle))

    def slice(self, begin: int, end: int) -> "Table":
        h = C.c_void_p()
        st = lib.ig_table_slice(self.handle, begin, end, C.byref(h))
        if st:
            _raise(st)
        return Table(h)

    def __del__(self):
        if getattr(self, "handle", None) and lib is not None:  # lib is None at interpreter teardown
            lib.ig_table_free(self.handle)
            self.handle = None


def read_csv(data: bytes) -> Table:
    h = C.c_void_p()
    st = lib.ig_read_csv(data, len(data), C.byref(h))
    if st:
        _raise(st)
    return Table(h)


class Schema:
    def __init__(self, handle, ncols):
        self.handle = handle
        self.ncols = ncols

    @property
    def label_index(self) -> int:
        return int(lib.ig_schema_label_index(self.handle))

    def column(self, j: int):
        kind, mean, sd = C.c_int(), C.c_double(), C.c_double()
        st = lib.ig_schema_column(self.handle, j, C.byref(kind), C.byref(mean), C.byref(sd))
        if st:
            _raise(st)
        return ("numeric" if kind.value == 0 else "categorical"), mean.value, sd.value

    def __del__(self):
        if getattr(self, "handle", None) and lib is not None:  # lib is None at interpreter teardown
            lib.ig_schema_free(self.handle)
            self.handle = None


def infer_schema(table: Table, label_column: str, attack_values=(), normal_values=(), decimals: int = 2) -> Schema:
    h = C.c_void_p()
    st = lib.ig_infer_schema(table.handle, label_column.encode(), ",".join(attack_values).encode(),
                             ",".join(normal_values).encode(), decimals, C.byref(h))
    if st:
        _raise(st)
    return Schema(h, table.columns)


class Columns:
    """Parsed, typed columns of a table under a schema (host; the fit's input)."""

    @classmethod
    def _wrap(cls, handle) -> "Columns":
        c = cls.__new__(cls)
        c.handle = handle
        return c

    def __init__(self, table: Table, schema: Schema, with_labels: bool = True):
        h = C.c_void_p()
        st = lib.ig_columns_build(table.handle, schema.handle, 1 if with_labels else 0, C.byref(h))
        if st:
            _raise(st)
        self.handle = h

    def upload(self, ctx: Optional[Context] = None) -> "Columns":
        ctx = ctx or default_context()
        ctx.check(lib.ig_columns_upload(ctx.handle, self.handle))
        return self

    def prefetch(self, ctx: Optional[Context] = None) -> "Columns":
        """Start the H2D copy now (copy stream); the next encode of these columns uses it."""
        ctx = ctx or default_context()
        ctx.check(lib.ig_columns_prefetch(ctx.handle, self.handle))
        return self

    @property
    def rows(self) -> int:
        return int(lib.ig_columns_rows(self.handle))

    @property
    def nbytes(self) -> int:
        return int(lib.ig_columns_bytes(self.handle))

    def __del__(self):
        if getattr(self, "handle", None) and lib is not None:  # lib is None at interpreter teardown
            lib.ig_columns_free(self.handle)
            self.handle = None


def ingest_csv(data: bytes, label_column: str = "label", attack_values=(), normal_values=(), decimals: int = 2,
               train_rows: Optional[int] = None, ratio_k: int = 8,
               ctx: Optional[Context] = None) -> tuple["Schema", "Columns", "Columns"]:
    """Device CSV ingest: (schema, train columns, test columns), resident on the
    device — the same as read_csv -> slice -> infer_schema -> Columns(...).upload.
    data: bytes, or a uint8 numpy array (e.g. pinned_array: the bytes then
    cross to the device at full copy-engine speed instead of being staged)."""
    ctx = ctx or default_context()
    hs, ht, he = C.c_void_p(), C.c_void_p(), C.c_void_p()
    if isinstance(data, np.ndarray):
        if data.dtype != np.uint8 or not data.flags.c_contiguous:
            raise ValueError("ingest_csv: a numpy input must be contiguous uint8")
        nbytes = int(data.size)
        data = C.cast(C.c_void_p(data.ctypes.data), C.c_char_p)
    else:
        nbytes = len(data)
    ctx.check(lib.ig_ingest_csv(ctx.handle, data, nbytes, label_column.encode(), ",".join(attack_values).encode(),
                                ",".join(normal_values).encode(), decimals,
                                -1 if train_rows is None else int(train_rows), ratio_k,
                                C.byref(hs), C.byref(ht), C.byref(he)))
    schema = Schema(hs, int(lib.ig_schema_cols(hs)))
    return schema, Columns._wrap(ht), Columns._wrap(he)


class Encoding:
    """Vocabulary + packed rows resident on the device (TrainingEncoding, pipeline.hpp:96-101)."""

    def __init__(self, ctx: Context, handle):
        self.ctx = ctx
        self.handle = handle

    @property
    def logical_len(self) -> int:
        return int(lib.ig_encoding_logical_len(self.handle))

    def rows(self, which: int) -> int:
        return int(lib.ig_encoding_rows(self.handle, which))

    def matrix(self, which: int) -> np.ndarray:
        n = self.rows(which)
        out = np.zeros((n, (self.logical_len + 63) // 64), np.int64)
        self.ctx.check(lib.ig_encoding_copy_rows(self.ctx.handle, self.handle, which, _p64(out)))
        return out

    def device_rows(self, which: int) -> int:
        return int(lib.ig_encoding_device_rows(self.handle, which) or 0)

    @property
    def vocabulary(self) -> list[str]:
        return lib.ig_encoding_vocabulary(self.handle).decode().split("\n")[:-1]

    @property
    def removed_rows(self) -> np.ndarray:
        n = lib.ig_encoding_removed_count(self.handle)
        out = np.zeros(n, np.uint64)
        if n:
            lib.ig_encoding_removed_rows(self.handle, out.ctypes.data_as(N.pu64))
        return out

    def __del__(self):
        if getattr(self, "handle", None) and lib is not None:  # lib is None at interpreter teardown
            lib.ig_encoding_free(self.handle)
            self.handle = None


def encode_training(columns: Columns, ctx: Optional[Context] = None) -> Encoding:
    ctx = ctx or default_context()
    h = C.c_void_p()
    ctx.check(lib.ig_encode_training(ctx.handle, columns.handle, C.byref(h)))
    return Encoding(ctx, h)


def encode_rows(columns: Columns, train: Encoding, ctx: Optional[Context] = None) -> Encoding:
    ctx = ctx or train.ctx
    h = C.c_void_p()
    ctx.check(lib.ig_encode_rows(ctx.handle, columns.handle, train.handle, C.byref(h)))
    return Encoding(ctx, h)


def fit_encoded(train: Encoding, config: Optional[KernelConfig] = None) -> Model:
    cfg = (config or KernelConfig()).c()
    h = C.c_void_p()
    train.ctx.check(lib.ig_fit_encoded(train.ctx.handle, train.handle, C.byref(cfg), C.byref(h)))
    return Model(train.ctx, h)


def fit_evidence_encoded(train: Encoding, tests: Encoding, config: Optional[KernelConfig] = None,
                         d_A_ptr: Optional[int] = None, d_N_ptr: Optional[int] = None):
    """fit + evidence of `tests` in one call (per-class overlap).  With device
    pointers the evidence lands there and only the Model is returned; otherwise
    (Model, A, N) with host arrays."""
    cfg = (config or KernelConfig()).c()
    h = C.c_void_p()
    if d_A_ptr is not None:
        train.ctx.check(lib.ig_fit_evidence_encoded(train.ctx.handle, train.handle, tests.handle, C.byref(cfg),
                                                    C.byref(h), C.c_void_p(d_A_ptr), C.c_void_p(d_N_ptr)))
        return Model(train.ctx, h)
    n = tests.rows(2)
    A = pinned_array((n,), np.int64)  # every element is written
    Nv = pinned_array((n,), np.int64)
    train.ctx.check(lib.ig_fit_evidence_encoded_host(train.ctx.handle, train.handle, tests.handle, C.byref(cfg),
                                                     C.byref(h), _p64(A), _p64(Nv)))
    return Model(train.ctx, h), A, Nv


# ---------------------------------------------------------------- infer / eval (host arithmetic)
def fit_normal_stats(nvals) -> tuple[float, float]:
    """mean / population std of strictly positive N; <2 positives -> (0, 0)
    (ig_fit_normal_stats: host C++, FMA-rounded like the reference's native build)."""
    nv = np.ascontiguousarray(nvals, np.int64)
    mu, sg = C.c_double(), C.c_double()
    st = lib.ig_fit_normal_stats(_p64(nv), nv.shape[0], C.byref(mu), C.byref(sg))
    if st:
        _raise(st)
    return mu.value, sg.value


def classify(A, Nv, mu: float, sigma: float, r: float = 0.568):
    """SPEC.md:444-452 (ig_classify). Returns (label, regulation) with regulation
    1 = R1-attack, 2 = R1-normal, 3 = R2, 4 = R3."""
    A = np.ascontiguousarray(A, np.int64)
    Nv = np.ascontiguousarray(Nv, np.int64)
    if A.shape != Nv.shape:
        raise ValueError("classify: A and N lengths differ")
    label = np.empty(A.shape[0], np.uint8)
    reg = np.empty(A.shape[0], np.uint8)
    st = lib.ig_classify(_p64(A), _p64(Nv), A.shape[0], float(mu), float(sigma), float(r),
                         label.ctypes.data_as(N.pu8), reg.ctypes.data_as(N.pu8))
    if st:
        _raise(st)
    return label, reg


def compute_metrics(pred, truth, margins) -> dict:
    """SPEC.md:518-526 (attack = positive; rank AUC with ties 0.5)."""
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
                balanced_auc=(rec + tnr) / 2, rank_auc=auc)


# ---------------------------------------------------------------- end to end (cmd_train + cmd_predict)
@dataclass
class RunResult:
    model: Model
    train: Encoding
    test: Optional[Encoding]
    A: Optional[np.ndarray]
    N: Optional[np.ndarray]


def train_and_score(csv: bytes, label_column: str = "label", decimals: int = 1, train_rows: Optional[int] = None,
                    ratio_k: int = 8, attack_values=(), normal_values=(), config: Optional[KernelConfig] = None,
                    ctx: Optional[Context] = None) -> RunResult:
    """split → schema → encode → fit → encode test → evidence."""
    ctx = ctx or default_context()
    table = read_csv(csv)
    n = table.rows
    ntr = train_rows if train_rows is not None else ratio_k * n // 10
    tr = table.slice(0, ntr)
    te = table.slice(ntr, n)
    schema = infer_schema(tr, label_column, attack_values, normal_values, decimals)
    ctr, cte = Columns(tr, schema, True), Columns(te, schema, False)
    ctr.prefetch(ctx)  # H2D on the copy stream: training columns first, test columns behind them
    if te.rows:
        cte.prefetch(ctx)
    enc = encode_training(ctr, ctx)
    if te.rows == 0:
        return RunResult(fit_encoded(enc, config), enc, None, None, None)
    tenc = encode_rows(cte, enc, ctx)
    model, A, Nv = fit_evidence_encoded(enc, tenc, config)
    return RunResult(model, enc, tenc, A, Nv)


# ---------------------------------------------------------------- archive / explain


def _esc(s: str) -> str:
    out = []
    for ch in s:
        o = ord(ch)
        out.append(f"\\x{o:02x}" if ch == "\\" or o < 0x20 else ch)
    return "".join(out)


def _unesc(s: str) -> str:
    out, i = [], 0
    while i < len(s):
        if s[i] == "\\" and s[i + 1:i + 2] == "x":
            out.append(chr(int(s[i + 2:i + 4], 16)))
            i += 4
        else:
            out.append(s[i])
            i += 1
    return "".join(out)


def schema_to_text(schema: Schema) -> str:
    n = C.c_size_t()
    st = lib.ig_schema_to_text(schema.handle, None, 0, C.byref(n))
    if st:
        _raise(st)
    buf = C.create_string_buffer(n.value + 1)
    lib.ig_schema_to_text(schema.handle, buf, n.value + 1, C.byref(n))
    return buf.raw[:n.value].decode("utf-8", errors="surrogateescape")


def schema_from_text(text: str) -> Schema:
    h = C.c_void_p()
    st = lib.ig_schema_from_text(text.encode("utf-8", errors="surrogateescape"), C.byref(h))
    if st:
        _raise(st)
    ncols = int(text.split("columns ", 1)[1].split("\n", 1)[0])
    return Schema(h, ncols)


def encoding_from_vocabulary(schema: Schema, vocabulary: list[str], ctx: Optional[Context] = None) -> Encoding:
    """The vocabulary lookup of a training encoding, rebuilt for test-time encode_rows."""
    ctx = ctx or default_context()
    blob = "".join(t + "\n" for t in vocabulary).encode("utf-8", errors="surrogateescape")
    h = C.c_void_p()
    st = lib.ig_encoding_from_vocabulary(schema.handle, blob, C.byref(h))
    if st:
        _raise(st)
    return Encoding(ctx, h)


def model_from_dictionaries(L: int, attack: Dictionary, normal: Dictionary, ctx: Optional[Context] = None) -> Model:
    ctx = ctx or default_context()
    arrs = []
    for d in (attack, normal):
        w = _words(d.words, L)
        s = np.ascontiguousarray(d.supports, np.int64)
        sc = np.ascontiguousarray(d.scores, np.int64)
        arrs.append((w, s, sc))
    h = C.c_void_p()
    (wa, sa, ca), (wn, sn, cn) = arrs
    ctx.check(lib.ig_model_from_dictionaries(ctx.handle, L, _p64(wa), _p64(sa), _p64(ca), wa.shape[0], _p64(wn),
                                             _p64(sn), _p64(cn), wn.shape[0], C.byref(h)))
    m = Model(ctx, h)
    m._keep = arrs
    return m


def explain(model: Model, row, cls: int) -> np.ndarray:
    """indices (ascending, into the pure dictionary of `cls`) of
    the patterns contained in one packed test row."""
    r = np.ascontiguousarray(row, np.int64).reshape(-1)
    cap = 1024
    while True:
        idx = np.zeros(cap, np.uint32)
        n = C.c_size_t()
        model.ctx.check(lib.ig_explain(model.ctx.handle, model.handle, cls, _p64(r), model.logical_len,
                                       idx.ctypes.data_as(C.POINTER(C.c_uint32)), cap, C.byref(n)))
        if n.value <= cap:
            return idx[:n.value].copy()
        cap = n.value


def explain_row(model: Model, row, vocabulary: list[str], dictionaries=None) -> dict:
    """Human-readable evidence of one row: matched pure patterns per class with
    their tokens, support and score; the score totals equal A and N."""
    dictionaries = dictionaries or [model.dictionary(0, 1), model.dictionary(1, 1)]
    out = {}
    for cls, name in ((0, "attack"), (1, "normal")):
        d = dictionaries[cls]
        items = []
        for i in explain(model, row, cls).tolist():
            words = d.words[i].view(np.uint64)
            toks = [vocabulary[w * 64 + b] for w in range(words.shape[0]) for b in range(64)
                    if (int(words[w]) >> b) & 1]
            items.append({"tokens": toks, "support": int(d.supports[i]), "score": int(d.scores[i])})
        out[name] = items
        out["A" if cls == 0 else "N"] = sum(x["score"] for x in items)
    return out


def save_model(model: Model, schema: Schema, vocabulary: list[str], r: float = 0.568,
               stats: Optional[tuple[float, float]] = None, provenance: str = "") -> bytes:
    """ModelArchive through ig_model_save: format_version,
    tool version, provenance, r, stats mode ("batch", or "frozen" with
    stats = (mu_N, sigma_N)), schema, vocabulary, both pure dictionaries;
    save -> load -> save is byte-identical."""
    blob = "".join(t + "\n" for t in vocabulary).encode("utf-8", errors="surrogateescape")
    prm = N.ArchiveParamsC(float(r), 1 if stats is not None else 0, float(stats[0]) if stats else 0.0,
                           float(stats[1]) if stats else 0.0,
                           provenance.encode("utf-8", errors="surrogateescape"))
    n = C.c_size_t()
    st = lib.ig_model_save(model.ctx.handle, model.handle, schema.handle, blob, C.byref(prm), None, 0, C.byref(n))
    if st:
        _raise(st)
    buf = C.create_string_buffer(n.value + 1)
    st = lib.ig_model_save(model.ctx.handle, model.handle, schema.handle, blob, C.byref(prm), buf, n.value + 1,
                           C.byref(n))
    if st:
        _raise(st)
    return buf.raw[:n.value]


@dataclass
class LoadedModel:
    model: Model
    schema: Schema
    vocabulary: list
    encoding: Encoding
    r: float
    stats: Optional[tuple[float, float]] = None  # frozen (mu_N, sigma_N), None = batch
    provenance: str = ""


def load_model(data: bytes, ctx: Optional[Context] = None) -> LoadedModel:
    """ig_model_load: the archive's model (evidence / explain ready), schema and
    the encoding that tokenises test rows like the training encoding."""
    ctx = ctx or default_context()
    cap = 1 << 16
    while True:
        hm, hs, he = C.c_void_p(), C.c_void_p(), C.c_void_p()
        prm = N.ArchiveParamsC()
        plen = C.c_size_t()
        pbuf = C.create_string_buffer(cap)
        st = lib.ig_model_load(ctx.handle, data, len(data), C.byref(hm), C.byref(hs), C.byref(he), C.byref(prm),
                               pbuf, cap, C.byref(plen))
        if st:
            _raise(st)
        model = Model(ctx, hm)
        schema = Schema(hs, int(lib.ig_schema_cols(hs)))
        enc = Encoding(ctx, he)
        if plen.value < cap:
            break
        cap = plen.value + 1  # provenance longer than the buffer: load again with room for it
    prov = pbuf.raw[:plen.value].decode("utf-8", errors="surrogateescape")
    return LoadedModel(model, schema, enc.vocabulary, enc, prm.r,
                       (prm.mu, prm.sigma) if prm.stats_frozen else None, prov)
