"""ctypes binding of libts_b200.so (include/ts_b200.h).

The library is built in-tree (``python -m paper_2601_16956_b200.build``) and
loaded from ``paper_2601_16956_b200/_lib``. There is no fallback: if the
library is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libts_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is not built; run `python -m paper_2601_16956_b200.build`")

lib = C.CDLL(LIB_PATH)

# --- status codes (ts_status) -------------------------------------------------
OK = 0
ERR_GENERIC, ERR_STREAM, ERR_CACHE_TIMEOUT, ERR_TICKET, ERR_TLV = 1, 2, 3, 4, 5
FORMAT_KINDS = {10: "missing_file", 11: "incomplete_file", 12: "corrupt_object", 13: "corrupt_footer",
                14: "bad_manifest", 15: "invalid_entries", 16: "io"}
ERR_CUDA, ERR_INVALID_ARG = 30, 31


class TsError(RuntimeError):
    """ts_error (common.hpp:21-24)."""

    def __init__(self, status: int, msg: str, object_id: int = -1):
        super().__init__(msg)
        self.status = status
        self.object_id = None if object_id < 0 else object_id


class StreamError(TsError):
    """stream_error{object_id} (provider.hpp:135-140)."""


class CacheTimeoutError(TsError):
    """cache_timeout_error (staging.hpp:18-21)."""


class TicketError(TsError):
    """ticket_error (transfer.hpp:41-44)."""


class TlvError(TsError):
    """tlv::tlv_error (tlv.hpp:70-73)."""


class FormatError(TsError):
    """format_error{kind, object_id} (format.hpp:50-67)."""

    @property
    def kind(self) -> str:
        return FORMAT_KINDS[self.status]


class CudaError(TsError):
    """CUDA failure or no device — the product has no CPU fallback."""


def raise_for(status: int):
    if status == OK:
        return
    msg = lib.ts_last_error().decode("utf-8", "replace")
    oid = lib.ts_last_error_object()
    cls = {ERR_STREAM: StreamError, ERR_CACHE_TIMEOUT: CacheTimeoutError, ERR_TICKET: TicketError,
           ERR_TLV: TlvError, ERR_CUDA: CudaError}.get(status)
    if cls is None:
        cls = FormatError if status in FORMAT_KINDS else TsError
    raise cls(status, msg, oid)


# --- structs ------------------------------------------------------------------


class ObjectDesc(C.Structure):
    _fields_ = [("object_id", C.c_uint64), ("kind", C.c_uint8), ("tier", C.c_uint8),
                ("precision", C.c_uint8), ("_pad", C.c_uint8), ("file_id", C.c_uint32),
                ("size_bytes", C.c_uint64), ("data", C.c_void_p), ("value", C.c_void_p)]


class RankInfo(C.Structure):
    _fields_ = [("rank_id", C.c_int32), ("tp_idx", C.c_int32), ("pp_idx", C.c_int32),
                ("dp_idx", C.c_int32)]


class FixedAssignment(C.Structure):
    _fields_ = [("object_id", C.c_uint64), ("file_offset", C.c_uint64), ("length", C.c_uint64)]


class EngineConfigC(C.Structure):
    _fields_ = [("strategy", C.c_int32), ("lazy_serialize_overlap", C.c_int32),
                ("staging_capacity_bytes", C.c_uint64), ("flush_workers", C.c_int32), ("_pad0", C.c_int32),
                ("raw_chunk_bytes", C.c_uint64), ("serialized_chunk_bytes", C.c_uint64),
                ("alignment", C.c_uint64), ("cache_acquire_timeout_ns", C.c_int64),
                ("overwrite", C.c_int32), ("d2h_mode", C.c_int32), ("device_staging_bytes", C.c_uint64),
                ("hybrid_direct_min_bytes", C.c_uint64), ("pack_ctas", C.c_int32),
                ("pack_threads", C.c_int32), ("pack_priority", C.c_int32), ("write_files", C.c_int32),
                ("checksum_on_gpu", C.c_int32), ("flush_mmap", C.c_int32), ("pack_kernel", C.c_int32),
                ("bulk_min_bytes", C.c_uint64), ("file_dma", C.c_int32), ("checksum_priority", C.c_int32),
                ("_pad2", C.c_int32), ("checksum_host_frac", C.c_double), ("ring_chunk_bytes", C.c_uint64),
                ("numa_bind", C.c_int32), ("worker_nice", C.c_int32),
                ("helper_mask", C.c_uint32), ("_pad4", C.c_uint32), ("helper_share", C.c_double),
                ("checksum_lane_max_bytes", C.c_int64)]


class ManifestEcho(C.Structure):
    _fields_ = [("tp", C.c_int32), ("pp", C.c_int32), ("dp", C.c_int32), ("zero1", C.c_int32),
                ("seed", C.c_uint64), ("n_params", C.c_uint64), ("layers", C.c_int32), ("_pad", C.c_int32),
                ("metadata_bytes", C.c_uint64)]


class TicketStats(C.Structure):
    _fields_ = [("checkpoint_id", C.c_uint64), ("total_bytes", C.c_uint64), ("raw_bytes", C.c_uint64),
                ("serialized_bytes", C.c_uint64), ("image_bytes", C.c_uint64),
                ("issue_block_ns", C.c_int64), ("barrier_block_ns", C.c_int64),
                ("t_captured_ns", C.c_int64), ("t_snapshot_ns", C.c_int64), ("t_persisted_ns", C.c_int64),
                ("pack_ms", C.c_float), ("d2h_ms", C.c_float), ("kernel_launches", C.c_uint32),
                ("copies", C.c_uint32), ("snapshot_done", C.c_int32), ("persisted_done", C.c_int32),
                ("failed", C.c_int32), ("file_dma_bytes", C.c_uint64),
                ("host_checksum_bytes", C.c_uint64), ("helper_bytes", C.c_uint64),
                ("direct_io_bytes", C.c_uint64), ("lane_checksum_bytes", C.c_uint64), ("lane_ms", C.c_float),
                ("_pad5", C.c_uint32), ("packed_bytes", C.c_uint64)]


class RestoreObject(C.Structure):
    _fields_ = [("object_id", C.c_uint64), ("kind", C.c_uint8), ("tier", C.c_uint8),
                ("precision", C.c_uint8), ("_pad", C.c_uint8), ("file_id", C.c_uint32),
                ("size_bytes", C.c_uint64)]


class RestoreStats(C.Structure):
    _fields_ = [("bytes", C.c_uint64), ("read_s", C.c_double), ("verify_s", C.c_double),
                ("h2d_unpack_s", C.c_double), ("total_s", C.c_double), ("unpack_ms", C.c_float),
                ("h2d_ms", C.c_float), ("kernel_launches", C.c_uint32), ("_pad", C.c_uint32),
                ("direct_bytes", C.c_uint64), ("direct_io_bytes", C.c_uint64)]


class VerifyIssue(C.Structure):
    _fields_ = [("kind", C.c_int32), ("_pad", C.c_int32), ("object_id", C.c_int64)]


class VerifyReportC(C.Structure):
    _fields_ = [("ok", C.c_int32), ("n_issues", C.c_int32), ("files_checked", C.c_uint64),
                ("objects_checked", C.c_uint64)]


class PatternDesc(C.Structure):
    _fields_ = [("data", C.c_void_p), ("size", C.c_uint64), ("space", C.c_uint64), ("offset", C.c_uint64)]


# --- signatures ---------------------------------------------------------------
P, u64, i64, i32, sz = C.c_void_p, C.c_uint64, C.c_int64, C.c_int, C.c_size_t


def _sig(name, res, *args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = list(args)


_sig("ts_last_error", C.c_char_p)
_sig("ts_last_error_object", i64)
_sig("ts_abi_version", i32)
for n in ("ts_value_null", "ts_value_list", "ts_value_map"):
    _sig(n, P)
_sig("ts_value_int", P, i64)
_sig("ts_value_float", P, C.c_double)
_sig("ts_value_string", P, C.c_char_p, sz)
_sig("ts_value_bytes", P, P, sz)
_sig("ts_value_list_append", i32, P, P)
_sig("ts_value_map_set", i32, P, C.c_char_p, sz, P)
_sig("ts_value_free", None, P)
_sig("ts_value_type", i32, P)
_sig("ts_value_as_int", i64, P)
_sig("ts_value_as_float", C.c_double, P)
_sig("ts_value_data", C.POINTER(C.c_uint8), P, C.POINTER(sz))
_sig("ts_value_len", sz, P)
_sig("ts_value_list_get", P, P, sz)
_sig("ts_value_map_key", P, P, sz, C.POINTER(sz), C.POINTER(C.c_char_p))
_sig("ts_value_encode", i32, P, P, sz, C.POINTER(sz))
_sig("ts_value_encoded_size", sz, P)
_sig("ts_value_decode", i32, P, sz, C.POINTER(P))
_sig("ts_make_metadata_value", P, i32, i32, i32, i32, u64, u64, u64)
_sig("ts_plan_layout", i32, C.POINTER(ObjectDesc), sz, u64, C.POINTER(C.c_uint32), C.POINTER(u64),
     C.POINTER(sz), C.POINTER(FixedAssignment), C.POINTER(C.c_uint32), C.POINTER(sz), C.POINTER(u64))
_sig("ts_fnv1a64", u64, P, sz, u64)
_sig("ts_engine_config_default", None, C.POINTER(EngineConfigC))
_sig("ts_engine_create", i32, C.POINTER(EngineConfigC), i32, i32, C.POINTER(P))
_sig("ts_engine_destroy", i32, P)
_sig("ts_retire_checkpoint", i32, C.c_char_p, C.c_char_p)
_sig("ts_engine_set_spare_dir", i32, P, C.c_char_p)
_sig("ts_engine_numa_node", i32, P)
_sig("ts_engine_provision_spares", i32, P, C.c_char_p, C.POINTER(RankInfo), C.POINTER(ObjectDesc), C.c_size_t,
     i32, C.POINTER(C.c_uint64))
_sig("ts_restore_set_file_cache", i32, P, i32)
_sig("ts_restore_set_direct_io", i32, P, i32)
_sig("ts_file_cache_bytes", C.c_uint64)
_sig("ts_file_cache_release_all", i32, C.POINTER(C.c_uint64))
_sig("ts_session_create", i32, C.c_char_p, u64, u64, C.POINTER(ManifestEcho), i32, i32, C.POINTER(P))
_sig("ts_session_destroy", i32, P)
_sig("ts_session_rank_blob", i32, P, i32, P, sz, C.POINTER(sz))
_sig("ts_session_add_remote_rank", i32, P, P, sz)
_sig("ts_session_register_rank", i32, P, C.POINTER(RankInfo), C.POINTER(ObjectDesc), sz)
_sig("ts_session_rank_persisted", i32, P, i32)
_sig("ts_session_wait_complete", i32, P, i64)
_sig("ts_session_complete", i32, P)
_sig("ts_issue", i32, P, P, C.POINTER(RankInfo), C.POINTER(ObjectDesc), sz, u64, P, C.POINTER(P))
_sig("ts_pre_update_barrier", i32, P, P, P, i32, C.POINTER(i64))
_sig("ts_ticket_wait_captured", i32, P, C.POINTER(i64))
_sig("ts_ticket_wait_snapshot", i32, P, C.POINTER(i64))
_sig("ts_ticket_wait_persisted", i32, P, C.POINTER(i64))
_sig("ts_ticket_stats_get", i32, P, C.POINTER(TicketStats))
_sig("ts_ticket_object_checksum", i32, P, u64, C.POINTER(u64))
_sig("ts_ticket_release", None, P)
_sig("ts_ticket_adopt_values", i32, P, C.POINTER(P), C.c_size_t)
_sig("ts_io_uring_available", i32)
_sig("ts_file_cache_stats", None, C.POINTER(u64))
_sig("ts_io_uring_ops", u64)
_sig("ts_restore_open", i32, C.c_char_p, C.POINTER(P))
_sig("ts_restore_close", None, P)
_sig("ts_restore_release_staging", C.c_uint64)
_sig("ts_restore_n_ranks", i32, P)
_sig("ts_restore_rank_info", i32, P, i32, C.POINTER(RankInfo))
_sig("ts_restore_rank_objects", i32, P, i32, C.POINTER(RestoreObject), sz, C.POINTER(sz))
_sig("ts_restore_rank", i32, P, i32, C.POINTER(ObjectDesc), sz, i32, P, C.POINTER(RestoreStats))
_sig("ts_restore_structured", i32, P, i32, u64, C.POINTER(P))
_sig("ts_verify", i32, C.c_char_p, C.POINTER(VerifyReportC), C.POINTER(VerifyIssue), sz)
_sig("ts_pattern_fill", i32, C.POINTER(PatternDesc), sz, u64, u64, P)
_sig("ts_pattern_verify", i32, C.POINTER(PatternDesc), sz, u64, u64, P, C.POINTER(u64))
_sig("ts_pack", i32, C.POINTER(P), C.POINTER(u64), C.POINTER(u64), sz, P, u64, i32, i32, P)
_sig("ts_unpack", i32, P, C.POINTER(u64), C.POINTER(P), C.POINTER(u64), sz, i32, i32, P)
_sig("ts_kernel_launch_count", u64)
_sig("ts_fnv1a64_device", i32, C.POINTER(P), C.POINTER(u64), sz, C.POINTER(u64), C.POINTER(u64), P)
_sig("ts_fnv1a64_device_lanes", i32, C.POINTER(P), C.POINTER(u64), sz, C.POINTER(u64), C.POINTER(u64), P)

def call(fn, *args):
    raise_for(fn(*args))
