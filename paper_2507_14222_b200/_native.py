"""ctypes binding of libig_b200.so (include/ig_b200.h).

The product path: there is no CPU fallback.  If the shared library is missing
this module raises at import time with the build command, so a GPU box without
the extension fails loudly instead of silently computing something else.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.environ.get("IG_B200_LIB") or os.path.join(HERE, "libig_b200.so")  # override: experiments only


class NativeMissing(ImportError):
    pass


def _load():
    if not os.path.exists(SO_PATH):
        raise NativeMissing(f"{SO_PATH} is not built: run `make -C {HERE}` (or __graft_entry__.build())")
    return C.CDLL(SO_PATH)


lib = _load()

p64 = C.POINTER(C.c_int64)
pu8 = C.POINTER(C.c_uint8)
pu64 = C.POINTER(C.c_uint64)
sz = C.c_size_t
vp = C.c_void_p
u32 = C.c_uint32


class ArchiveParamsC(C.Structure):
    _fields_ = [("r", C.c_double), ("stats_frozen", C.c_int), ("mu", C.c_double), ("sigma", C.c_double),
                ("provenance", C.c_char_p)]


class KernelConfigC(C.Structure):
    _fields_ = [("pair_batch", sz), ("coverage_block", sz), ("memory_budget_bytes", sz), ("threads", C.c_int)]


PROGRESS = C.CFUNCTYPE(None, C.c_uint64, C.c_uint64, C.c_uint64, vp)

# (name, restype, argtypes) — every symbol declared in include/ig_b200.h
SIGNATURES = [
    ("ig_ctx_create", C.c_int, [C.c_int, C.POINTER(vp)]),
    ("ig_ctx_destroy", None, [vp]),
    ("ig_last_error", C.c_char_p, [vp]),
    ("ig_ctx_set_stream", C.c_int, [vp, vp]),
    ("ig_ctx_launch_count", C.c_uint64, [vp]),
    ("ig_version", C.c_char_p, []),
    ("ig_ctx_set_diagnostics", C.c_int, [vp, C.c_int]),
    ("ig_ctx_diag_kernel", C.c_int, [vp, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_uint64),
                               C.POINTER(C.c_uint64)]),
    ("ig_measure_int_peaks", C.c_int, [vp, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    ("ig_kernel_config_default", None, [C.POINTER(KernelConfigC)]),
    ("ig_pair_intersect_batch", C.c_int, [vp, p64, sz, u32, sz, sz, sz, p64]),
    ("ig_coverage_any", C.c_int, [vp, p64, sz, u32, p64, sz, u32, sz, pu8]),
    ("ig_fused_score", C.c_int, [vp, p64, sz, u32, p64, sz, p64, sz, u32, p64]),
    ("ig_enumerate_candidates", C.c_int, [vp, p64, sz, u32, C.POINTER(KernelConfigC), PROGRESS, vp, C.POINTER(vp)]),
    ("ig_count_support", C.c_int, [vp, vp, p64, sz, u32, C.POINTER(KernelConfigC)]),
    ("ig_count_support_rows", C.c_int, [vp, p64, sz, u32, p64, sz, u32, p64]),
    ("ig_score_patterns", C.c_int, [vp, vp]),
    ("ig_total_score", C.c_int, [p64, sz, p64]),
    ("ig_fit_normal_stats", C.c_int, [p64, sz, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    ("ig_classify", C.c_int, [p64, p64, sz, C.c_double, C.c_double, C.c_double, pu8, pu8]),
    ("ig_candidates_count", sz, [vp]),
    ("ig_candidates_logical_len", u32, [vp]),
    ("ig_candidates_copy", C.c_int, [vp, vp, p64, p64, p64]),
    ("ig_candidates_free", None, [vp]),
    ("ig_fit", C.c_int, [vp, p64, sz, p64, sz, u32, C.POINTER(KernelConfigC), C.POINTER(vp)]),
    ("ig_fit_device", C.c_int, [vp, vp, sz, vp, sz, u32, C.POINTER(KernelConfigC), C.POINTER(vp)]),
    ("ig_model_count", sz, [vp, C.c_int, C.c_int]),
    ("ig_model_logical_len", u32, [vp]),
    ("ig_model_copy", C.c_int, [vp, vp, C.c_int, C.c_int, p64, p64, p64]),
    ("ig_model_phase_ms", C.c_int, [vp, C.POINTER(C.c_double)]),
    ("ig_host_alloc", C.c_int, [sz, C.POINTER(vp)]),
    ("ig_host_free", None, [vp]),
    ("ig_model_free", None, [vp]),
    ("ig_evidence", C.c_int, [vp, vp, p64, sz, u32, p64, p64]),
    ("ig_evidence_device", C.c_int, [vp, vp, vp, sz, u32, vp, vp]),
    ("ig_read_csv", C.c_int, [C.c_char_p, sz, C.POINTER(vp)]),
    ("ig_table_rows", sz, [vp]),
    ("ig_table_cols", sz, [vp]),
    ("ig_table_slice", C.c_int, [vp, sz, sz, C.POINTER(vp)]),
    ("ig_table_free", None, [vp]),
    ("ig_infer_schema", C.c_int, [vp, C.c_char_p, C.c_char_p, C.c_char_p, C.c_int, C.POINTER(vp)]),
    ("ig_schema_column", C.c_int, [vp, sz, C.POINTER(C.c_int), C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    ("ig_schema_label_index", sz, [vp]),
    ("ig_schema_cols", sz, [vp]),
    ("ig_schema_free", None, [vp]),
    ("ig_columns_build", C.c_int, [vp, vp, C.c_int, C.POINTER(vp)]),
    ("ig_columns_upload", C.c_int, [vp, vp]),
    ("ig_columns_prefetch", C.c_int, [vp, vp]),
    ("ig_ingest_csv", C.c_int, [vp, C.c_char_p, sz, C.c_char_p, C.c_char_p, C.c_char_p, C.c_int, C.c_longlong,
                                C.c_int, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp)]),
    ("ig_columns_rows", sz, [vp]),
    ("ig_columns_bytes", sz, [vp]),
    ("ig_columns_free", None, [vp]),
    ("ig_encode_training", C.c_int, [vp, vp, C.POINTER(vp)]),
    ("ig_encode_rows", C.c_int, [vp, vp, vp, C.POINTER(vp)]),
    ("ig_encoding_logical_len", u32, [vp]),
    ("ig_encoding_rows", sz, [vp, C.c_int]),
    ("ig_encoding_device_rows", vp, [vp, C.c_int]),
    ("ig_encoding_copy_rows", C.c_int, [vp, vp, C.c_int, p64]),
    ("ig_encoding_vocabulary", C.c_char_p, [vp]),
    ("ig_encoding_removed_count", sz, [vp]),
    ("ig_encoding_removed_rows", C.c_int, [vp, pu64]),
    ("ig_encoding_free", None, [vp]),
    ("ig_fit_encoded", C.c_int, [vp, vp, C.POINTER(KernelConfigC), C.POINTER(vp)]),
    ("ig_schema_to_text", C.c_int, [vp, C.c_char_p, sz, C.POINTER(sz)]),
    ("ig_schema_from_text", C.c_int, [C.c_char_p, C.POINTER(vp)]),
    ("ig_encoding_from_vocabulary", C.c_int, [vp, C.c_char_p, C.POINTER(vp)]),
    ("ig_model_from_dictionaries", C.c_int, [vp, u32, p64, p64, p64, sz, p64, p64, p64, sz, C.POINTER(vp)]),
    ("ig_model_save", C.c_int, [vp, vp, vp, C.c_char_p, C.POINTER(ArchiveParamsC), C.c_char_p, sz, C.POINTER(sz)]),
    ("ig_model_load", C.c_int, [vp, C.c_char_p, sz, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp),
                                C.POINTER(ArchiveParamsC), C.c_char_p, sz, C.POINTER(sz)]),
    ("ig_explain", C.c_int, [vp, vp, C.c_int, p64, u32, C.POINTER(C.c_uint32), sz, C.POINTER(sz)]),
    ("ig_shard_create", C.c_int, [vp, vp, C.c_int, C.c_int, C.POINTER(KernelConfigC), C.POINTER(vp)]),
    ("ig_shard_enumerate", C.c_int, [vp, vp, C.c_int, pu64, C.POINTER(vp)]),
    ("ig_shard_receive", C.c_int, [vp, vp, C.c_int, vp, C.c_uint64]),
    ("ig_shard_finish", C.c_int, [vp, vp, pu64]),
    ("ig_shard_model", vp, [vp]),
    ("ig_shard_free", None, [vp]),
    ("ig_evidence_encoded", C.c_int, [vp, vp, vp, p64, p64]),
    ("ig_evidence_encoded_device", C.c_int, [vp, vp, vp, vp, vp]),
    ("ig_fit_evidence_encoded", C.c_int, [vp, vp, vp, vp, C.POINTER(vp), vp, vp]),
    ("ig_fit_evidence_encoded_host", C.c_int, [vp, vp, vp, vp, C.POINTER(vp), p64, p64]),
]

for _name, _res, _args in SIGNATURES:
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args
