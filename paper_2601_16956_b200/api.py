"""Python mirror of the reference's State Provider / checkpoint-engine API on top
of the C-ABI (include/ts_b200.h).

Names, argument meaning and error behaviour follow the reference
(/root/reference/proj): ``StateObject``/``RankState`` (model.hpp:34-73),
``EngineConfig`` (engine.hpp:34-52), ``CheckpointSession`` (engine.hpp:57-90),
``CheckpointEngine.issue_checkpoint`` / ``pre_update_barrier``
(engine.hpp:107-113), ``TransferTicket`` (transfer.hpp:52-88),
``restore_checkpoint`` / ``verify_checkpoint`` (format.hpp:161-178), and the
synthetic-state helpers ``materialize_payloads`` / ``mutate_update_step``
(model.hpp:123-130). Raw payloads are CUDA tensors; every byte they hold is
moved by this library's kernels / DMA, never by PyTorch.
"""
from __future__ import annotations

import ctypes as C
import struct
import os
from dataclasses import dataclass, field
from typing import Any, Dict, List, Optional

import torch

from . import _native as N

try:  # CPython fast path of _desc_array (built next to libts_b200.so by build.py)
    from . import _pyfast
except ImportError:  # pragma: no cover - the pure-Python path is complete, only slower
    _pyfast = None
from .synthetic import Recipe, RankSpec

TIER_DEVICE, TIER_HOST, TIER_PERSISTENT = 0, 1, 2
KIND_RAW, KIND_STRUCTURED = 0, 1
STRATEGY = {"sync": 0, "two_phase": 1, "lazy": 2}
D2H_MODE = {"ring": 0, "direct": 1, "zerocopy": 2, "hybrid": 3}

TsError, StreamError, CacheTimeoutError, TicketError, TlvError, FormatError, CudaError = (
    N.TsError, N.StreamError, N.CacheTimeoutError, N.TicketError, N.TlvError, N.FormatError, N.CudaError)


# ---------------------------------------------------------------------------
# TLV values (tlv.hpp:24-83)


class Value:
    """Owning handle of a native TLV value."""

    __slots__ = ("h",)

    def __init__(self, h: int):
        if not h:
            raise TsError(N.ERR_GENERIC, "null value handle")
        self.h = h

    def __del__(self, _free=N.lib.ts_value_free):
        h, self.h = getattr(self, "h", None), None
        if h:
            _free(h)

    @staticmethod
    def from_py(v: Any) -> "Value":
        # Fast path: canonical TLV bytes built in Python, one native decode
        # (strict: invalid UTF-8, depth > 256 are rejected there). Anything
        # unusual takes the element-by-element native builder.
        try:
            out = bytearray()
            _enc_py(v, out, 0)
            return Value.decode(bytes(out))
        except (_Fallback, TsError):
            return Value(_build(v))

    @staticmethod
    def metadata(rank_id, tp_idx, pp_idx, dp_idx, seed, metadata_bytes, iteration) -> "Value":
        """make_metadata_value (model.cpp:206-231), built natively."""
        return Value(N.lib.ts_make_metadata_value(rank_id, tp_idx, pp_idx, dp_idx, seed & (2**64 - 1),
                                                  metadata_bytes, iteration))

    def encode(self) -> bytes:
        n = N.lib.ts_value_encoded_size(self.h)
        buf = (C.c_uint8 * max(1, n))()
        ln = C.c_size_t()
        N.call(N.lib.ts_value_encode, self.h, buf, n, C.byref(ln))
        return bytes(buf)[:ln.value]

    @staticmethod
    def decode(data: bytes) -> "Value":
        out = C.c_void_p()
        N.call(N.lib.ts_value_decode, data, len(data), C.byref(out))
        return Value(out.value)

    def to_py(self) -> Any:
        return _to_py(self.h)


class _Fallback(Exception):
    pass


_U64 = struct.Struct("<Q")
_I64 = struct.Struct("<q")
_F64 = struct.Struct("<d")


def _enc_py(v: Any, out: bytearray, depth: int) -> None:
    """tlv::encode (tlv.cpp:39-77) of a plain Python value: tags 0 null,
    1 int64, 2 f64, 3 utf8, 4 bytes, 5 list, 6 map (keys sorted, tagged strings)."""
    if depth > 200:
        raise _Fallback
    if v is None:
        out.append(0)
    elif isinstance(v, bool):
        raise _Fallback
    elif isinstance(v, int):
        if not -2**63 <= v < 2**64:
            raise _Fallback
        out.append(1)
        out += _I64.pack(v if v < 2**63 else v - 2**64)
    elif isinstance(v, float):
        out.append(2)
        out += _F64.pack(v)
    elif isinstance(v, str):
        try:
            b = v.encode("utf-8")
        except UnicodeEncodeError:
            raise _Fallback
        out.append(3)
        out += _U64.pack(len(b))
        out += b
    elif isinstance(v, (bytes, bytearray, memoryview)):
        b = bytes(v)
        out.append(4)
        out += _U64.pack(len(b))
        out += b
    elif isinstance(v, (list, tuple)):
        out.append(5)
        out += _U64.pack(len(v))
        for x in v:
            _enc_py(x, out, depth + 1)
    elif isinstance(v, dict):
        items = []
        for k, x in v.items():
            try:
                items.append((str(k).encode("utf-8"), x))
            except UnicodeEncodeError:
                raise _Fallback
        items.sort(key=lambda kv: kv[0])
        if any(items[i][0] == items[i + 1][0] for i in range(len(items) - 1)):
            raise _Fallback
        out.append(6)
        out += _U64.pack(len(items))
        for kb, x in items:
            out.append(3)
            out += _U64.pack(len(kb))
            out += kb
            _enc_py(x, out, depth + 1)
    else:
        raise _Fallback


def _build(v: Any) -> int:
    L = N.lib
    if isinstance(v, Value):
        return _clone(v)
    if v is None:
        return L.ts_value_null()
    if isinstance(v, bool):
        raise TlvError(N.ERR_TLV, "bool is not a TLV type")
    if isinstance(v, int):
        return L.ts_value_int(C.c_int64(v if v < 2**63 else v - 2**64))
    if isinstance(v, float):
        return L.ts_value_float(v)
    if isinstance(v, str):
        b = v.encode("utf-8", "surrogatepass")
        return L.ts_value_string(b, len(b))
    if isinstance(v, (bytes, bytearray, memoryview)):
        b = bytes(v)
        return L.ts_value_bytes(b, len(b))
    if hasattr(v, "tobytes") and not isinstance(v, torch.Tensor):
        b = v.tobytes()
        return L.ts_value_bytes(b, len(b))
    if isinstance(v, (list, tuple)):
        h = L.ts_value_list()
        for x in v:
            N.call(L.ts_value_list_append, h, _build(x))
        return h
    if isinstance(v, dict):
        h = L.ts_value_map()
        for k, x in v.items():
            kb = str(k).encode("utf-8")
            N.call(L.ts_value_map_set, h, kb, len(kb), _build(x))
        return h
    raise TlvError(N.ERR_TLV, f"unsupported type {type(v)}")


def _clone(v: Value) -> int:
    enc = v.encode()
    out = C.c_void_p()
    N.call(N.lib.ts_value_decode, enc, len(enc), C.byref(out))
    return out.value


def _to_py(h: int) -> Any:
    L = N.lib
    t = L.ts_value_type(h)
    if t == 0:
        return None
    if t == 1:
        return L.ts_value_as_int(h)
    if t == 2:
        return L.ts_value_as_float(h)
    if t in (3, 4):
        n = C.c_size_t()
        p = L.ts_value_data(h, C.byref(n))
        b = C.string_at(p, n.value) if n.value else b""
        return b.decode("utf-8") if t == 3 else b
    if t == 5:
        return [_to_py(L.ts_value_list_get(h, i)) for i in range(L.ts_value_len(h))]
    if t == 6:
        out = {}
        for i in range(L.ts_value_len(h)):
            kn, kp = C.c_size_t(), C.c_char_p()
            x = L.ts_value_map_key(h, i, C.byref(kn), C.byref(kp))
            out[C.string_at(kp, kn.value).decode("utf-8")] = _to_py(x)
        return out
    raise TlvError(N.ERR_TLV, "bad value handle")


def tlv_encode(v: Any) -> bytes:
    return Value.from_py(v).encode()


def tlv_decode(b: bytes) -> Any:
    return Value.decode(b).to_py()


def fnv1a64_device(tensors, init=None, stream=None, lanes=False):
    """FNV-1a-64 of each device tensor's bytes, computed by the GPU kernels
    (segment-parallel; lanes=True: the lane-serial kernel)."""
    n = len(tensors)
    ptrs = (C.c_void_p * max(1, n))(*[t.data_ptr() for t in tensors])
    sizes = (C.c_uint64 * max(1, n))(*[t.numel() * t.element_size() for t in tensors])
    out = (C.c_uint64 * max(1, n))()
    ini = (C.c_uint64 * max(1, n))(*init) if init is not None else None
    sh = _stream_handle(stream)
    fn = N.lib.ts_fnv1a64_device_lanes if lanes else N.lib.ts_fnv1a64_device
    N.call(fn, ptrs, sizes, n, ini, out, C.c_void_p(sh))
    return list(out)[:n]


def fnv1a64(data, state: int = 14695981039346656037) -> int:
    """FNV-1a-64 (common.hpp:44-51) of host bytes."""
    b = bytes(data)
    return N.lib.ts_fnv1a64(b, len(b), state)


# ---------------------------------------------------------------------------
# State model (model.hpp:34-73)


@dataclass
class StateObject:
    object_id: int
    kind: int = KIND_RAW
    residency: int = TIER_DEVICE
    precision: int = 2
    file_id: int = 0
    size_bytes: int = 0
    pattern_space: int = 0
    pattern_offset: int = 0
    payload: Optional[torch.Tensor] = None   # raw: tensor holding exactly size_bytes bytes
    structured: Any = None                   # structured: python value or Value

    def is_raw(self) -> bool:
        return self.kind == KIND_RAW


@dataclass
class RankState:
    rank_id: int = 0
    tp_idx: int = 0
    pp_idx: int = 0
    dp_idx: int = 0
    seed: int = 0
    metadata_bytes: int = 0
    objects: List[StateObject] = field(default_factory=list)
    arena: Optional[torch.Tensor] = None      # flat device buffer the raw shards are views of

    def raw_bytes(self) -> int:
        return sum(o.size_bytes for o in self.objects if o.is_raw())

    @property
    def file_ids(self) -> List[int]:
        return sorted({o.file_id for o in self.objects})


def _desc_array(rank: RankState, keep: list, need_payload: bool = True):
    arr = (N.ObjectDesc * max(1, len(rank.objects)))()
    if _pyfast is not None:
        # one C walk over the objects (csrc/pyfast); anything it does not take
        # (unusual values, errors) goes the pure-Python way below
        try:
            _pyfast.fill_descs(rank.objects, C.addressof(arr), need_payload, Value, keep)
            return arr
        except Exception:
            C.memset(arr, 0, C.sizeof(arr))
            keep.clear()
    for i, o in enumerate(rank.objects):
        d = arr[i]
        d.object_id, d.kind, d.tier, d.precision, d.file_id = (o.object_id, o.kind, o.residency,
                                                               o.precision, o.file_id)
        if o.is_raw():
            d.size_bytes = o.size_bytes
            if o.payload is not None:
                d.data = o.payload.data_ptr()
            elif need_payload:
                raise TsError(N.ERR_GENERIC, "raw source: payload not materialized")
        elif need_payload:
            v = o.structured if isinstance(o.structured, Value) else Value.from_py(o.structured)
            keep.append(v)
            d.value = v.h
    return arr


# ---------------------------------------------------------------------------
# Engine (engine.hpp:34-153)


@dataclass
class EngineConfig:
    strategy: str = "lazy"
    lazy_serialize_overlap: bool = True
    staging_capacity_bytes: int = 256 << 20
    flush_workers: int = 4
    raw_chunk_bytes: int = 16 << 20
    serialized_chunk_bytes: int = 1 << 20
    alignment: int = 4096
    cache_acquire_timeout_ns: Optional[int] = 300 * 10**9
    overwrite: bool = True
    # B200 knobs
    d2h_mode: str = "hybrid"  # = ring when the image fits the device staging (full shadow)
    device_staging_bytes: int = 2 << 30
    hybrid_direct_min_bytes: int = 1 << 20  # HYBRID head only if its mean fragment piece is >= this
    pack_ctas: int = 0
    pack_threads: int = 512
    pack_priority: int = 1  # capture stream: 1 high (default), 0 normal, -1 low
    write_files: bool = True
    checksum_on_gpu: bool = True
    flush_mmap: int = 1  # 1: copy into a shared mapping; 0: pwrite; 2: O_DIRECT body + pwrite head/tail; 3: 2 via io_uring
    pack_kernel: str = "bulk"  # "bulk" (TMA cp.async.bulk for large aligned fragments + warp kernel) | "warp"
    #                          | "bulk-ring" (also in a multi-slot ring, 2-stage / 64 KiB kernel)
    bulk_min_bytes: int = 1 << 20
    file_dma: bool = True  # D2H straight into page-locked file pages when registered (rotation)
    checksum_priority: int = -1  # RING device checksums' stream: 1 high, 0 normal, -1 low (default)
    checksum_host_frac: float = -1.0  # share hashed by host workers: 0 all GPU, <0 auto (default)
    ring_chunk_bytes: int = 0  # RING slot size without a full shadow (0 = auto: ring/6, <= 8 GiB)
    numa_bind: bool = True  # engine threads + pinned pool on the GPU's NUMA node (multi-socket hosts)
    worker_nice: int = 19  # nice increment of the background worker threads (0 = none)
    helper_devices: tuple = ()  # RING: GPUs whose copy engines carry part of this rank's D2H (NVLink read)
    helper_share: float = 0.0  # fraction of the image they carry
    checksum_lane_max_bytes: int = 0  # lane-serial FNV for objects up to this size (0 off, -1 auto)

    def to_c(self) -> N.EngineConfigC:
        c = N.EngineConfigC()
        N.lib.ts_engine_config_default(C.byref(c))
        c.strategy = STRATEGY[self.strategy]
        c.lazy_serialize_overlap = int(self.lazy_serialize_overlap)
        c.staging_capacity_bytes = self.staging_capacity_bytes
        c.flush_workers = self.flush_workers
        c.raw_chunk_bytes = self.raw_chunk_bytes
        c.serialized_chunk_bytes = self.serialized_chunk_bytes
        c.alignment = self.alignment
        c.cache_acquire_timeout_ns = -1 if self.cache_acquire_timeout_ns is None else self.cache_acquire_timeout_ns
        c.overwrite = int(self.overwrite)
        c.d2h_mode = D2H_MODE[self.d2h_mode]
        c.device_staging_bytes = self.device_staging_bytes
        c.hybrid_direct_min_bytes = self.hybrid_direct_min_bytes
        c.pack_ctas = self.pack_ctas
        c.pack_threads = self.pack_threads
        c.pack_priority = int(self.pack_priority)
        c.write_files = int(self.write_files)
        c.checksum_on_gpu = int(self.checksum_on_gpu)
        c.flush_mmap = int(self.flush_mmap)
        c.pack_kernel = {"warp": 0, "bulk": 1, "bulk-ring": 2}[self.pack_kernel]
        c.bulk_min_bytes = self.bulk_min_bytes
        c.file_dma = int(self.file_dma)
        c.checksum_priority = int(self.checksum_priority)
        c.checksum_host_frac = float(self.checksum_host_frac)
        c.ring_chunk_bytes = int(self.ring_chunk_bytes)
        c.numa_bind = int(self.numa_bind)
        c.worker_nice = int(self.worker_nice)
        c.helper_mask = sum(1 << int(d) for d in self.helper_devices)
        c.helper_share = float(self.helper_share)
        c.checksum_lane_max_bytes = int(self.checksum_lane_max_bytes)
        return c


class CheckpointSession:
    """checkpoint_session: commit scope of one checkpoint; MANIFEST.tlv is written
    last, by the process with writes_manifest=True, once n_ranks ranks persisted."""

    def __init__(self, dir: str, checkpoint_id: int, iteration: int, layout_echo: Optional[dict] = None,
                 n_ranks: int = 1, writes_manifest: bool = True):
        self.dir = dir
        self.checkpoint_id = checkpoint_id
        self.iteration = iteration
        echo = None
        if layout_echo:
            echo = N.ManifestEcho(layout_echo["tp"], layout_echo["pp"], layout_echo["dp"], layout_echo["zero1"],
                                  layout_echo["seed"], layout_echo["n_params"], layout_echo["layers"], 0,
                                  layout_echo["metadata_bytes"])
        h = C.c_void_p()
        N.call(N.lib.ts_session_create, dir.encode(), checkpoint_id, iteration,
               C.byref(echo) if echo is not None else None, n_ranks, int(writes_manifest), C.byref(h))
        self.h = h.value

    @property
    def manifest_path(self) -> str:
        return os.path.join(self.dir, "MANIFEST.tlv")

    def rank_blob(self, rank_id: int) -> bytes:
        n = C.c_size_t()
        N.lib.ts_session_rank_blob(self.h, rank_id, None, 0, C.byref(n))
        buf = (C.c_uint8 * max(1, n.value))()
        N.call(N.lib.ts_session_rank_blob, self.h, rank_id, buf, n.value, C.byref(n))
        return bytes(buf)[:n.value]

    def add_remote_rank(self, blob: bytes):
        N.call(N.lib.ts_session_add_remote_rank, self.h, blob, len(blob))

    def register_rank(self, rank: RankState):
        """Manifest info of a rank checkpointed by another engine/process."""
        keep: list = []
        arr = _desc_array(rank, keep, need_payload=False)
        info = N.RankInfo(rank.rank_id, rank.tp_idx, rank.pp_idx, rank.dp_idx)
        N.call(N.lib.ts_session_register_rank, self.h, C.byref(info), arr, len(rank.objects))

    def rank_persisted(self, rank_id: int):
        N.call(N.lib.ts_session_rank_persisted, self.h, rank_id)

    def wait_complete(self, timeout_s: Optional[float] = None):
        N.call(N.lib.ts_session_wait_complete, self.h, -1 if timeout_s is None else int(timeout_s * 1e9))

    @property
    def complete(self) -> bool:
        return bool(N.lib.ts_session_complete(self.h))

    def close(self):
        if self.h:
            N.call(N.lib.ts_session_destroy, self.h)
            self.h = None


class TransferTicket:
    """transfer_ticket: per-(checkpoint, rank) progress handle."""

    def __init__(self, h: int, keep: list):
        self.h = h
        self._keep = keep  # structured values the serializers still read

    def __del__(self, _wait=N.lib.ts_ticket_wait_snapshot, _rel=N.lib.ts_ticket_release):
        h, self.h = getattr(self, "h", None), None
        if h:
            try:
                _wait(h, None)  # serializers hold raw pointers to _keep
            finally:
                _rel(h)

    def _wait(self, fn) -> int:
        ns = C.c_int64()
        N.call(fn, self.h, C.byref(ns))
        return ns.value

    def wait_captured(self) -> int:
        """State may be mutated (device-side copy complete)."""
        return self._wait(N.lib.ts_ticket_wait_captured)

    def wait_snapshot(self) -> int:
        return self._wait(N.lib.ts_ticket_wait_snapshot)

    def wait_persisted(self) -> int:
        return self._wait(N.lib.ts_ticket_wait_persisted)

    def stats(self) -> Dict[str, Any]:
        s = N.TicketStats()
        N.call(N.lib.ts_ticket_stats_get, self.h, C.byref(s))
        return {f: getattr(s, f) for f, _ in N.TicketStats._fields_}

    @property
    def snapshot_done(self) -> bool:
        return bool(self.stats()["snapshot_done"])

    @property
    def persisted_done(self) -> bool:
        return bool(self.stats()["persisted_done"])

    @property
    def issue_block_ns(self) -> int:
        return self.stats()["issue_block_ns"]

    @property
    def barrier_block_ns(self) -> int:
        return self.stats()["barrier_block_ns"]

    def object_checksum(self, object_id: int) -> int:
        out = C.c_uint64()
        N.call(N.lib.ts_ticket_object_checksum, self.h, object_id, C.byref(out))
        return out.value


def _stream_handle(stream) -> int:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


class CheckpointEngine:
    """checkpoint_engine for one rank on one GPU."""

    def __init__(self, config: Optional[EngineConfig] = None, rank_id: int = 0, device: int = 0):
        self.config = config or EngineConfig()
        self.rank_id = rank_id
        self.device = device
        c = self.config.to_c()
        h = C.c_void_p()
        N.call(N.lib.ts_engine_create, C.byref(c), rank_id, device, C.byref(h))
        self.h = h.value

    def issue_checkpoint(self, session: CheckpointSession, rank: RankState, iteration: int,
                         producer_stream=None) -> TransferTicket:
        keep: list = []
        arr = _desc_array(rank, keep)
        info = N.RankInfo(rank.rank_id, rank.tp_idx, rank.pp_idx, rank.dp_idx)
        out = C.c_void_p()
        with torch.cuda.device(self.device):
            sh = _stream_handle(producer_stream)
        N.call(N.lib.ts_issue, self.h, session.h, C.byref(info), arr, len(rank.objects), iteration,
               C.c_void_p(sh), C.byref(out))
        return TransferTicket(out.value, keep)

    def pre_update_barrier(self, ticket: Optional[TransferTicket], stream=None, host_block: int = 1) -> int:
        """host_block: 0 = the optimizer stream waits on the capture (no host block);
        1 = the host waits for the capture; 2 = the host waits for the whole
        snapshot (reference wait_snapshot semantics, engine.cpp:621-630)."""
        if ticket is None:
            return 0
        ns = C.c_int64()
        with torch.cuda.device(self.device):
            sh = _stream_handle(stream)
        N.call(N.lib.ts_pre_update_barrier, self.h, ticket.h, C.c_void_p(sh), host_block, C.byref(ns))
        return ns.value

    @property
    def numa_node(self) -> int:
        """NUMA node of the engine's threads and pinned pool (-1: none / single node)."""
        return int(N.lib.ts_engine_numa_node(self.h))

    def provision_spares(self, spare_dir: str, rank: RankState, copies: int = 2) -> int:
        """Spare files for this rank's layout in `spare_dir`, page-locked ahead of
        time: with rotation, even the first checkpoints take the direct D2H.
        Returns the bytes locked."""
        keep: list = []
        arr = _desc_array(rank, keep, need_payload=False)
        info = N.RankInfo(rank.rank_id, rank.tp_idx, rank.pp_idx, rank.dp_idx)
        out = C.c_uint64(0)
        N.call(N.lib.ts_engine_provision_spares, self.h, spare_dir.encode(), C.byref(info), arr,
               len(rank.objects), int(copies), C.byref(out))
        return int(out.value)

    def set_spare_dir(self, spare_dir: str):
        """Take over files of checkpoints retired into `spare_dir` (retire_checkpoint)."""
        N.call(N.lib.ts_engine_set_spare_dir, self.h, spare_dir.encode())

    def shutdown(self):
        if self.h:
            N.call(N.lib.ts_engine_destroy, self.h)
            self.h = None

    def __del__(self):
        try:
            self.shutdown()
        except Exception:
            pass


# ---------------------------------------------------------------------------
# Synthetic state on the GPU (model.cpp:195-244)


def _align(v: int, a: int) -> int:
    return (v + a - 1) // a * a


def materialize_payloads(spec: RankSpec, device: int = 0, iteration: int = 0, stream=None,
                         arena: Optional[torch.Tensor] = None) -> RankState:
    """Allocates the rank's raw objects as views of one flat HBM buffer (each shard
    at its own alignment, like ZeRO flat partitions) and fills them with
    pattern(seed, space, iteration) on the GPU."""
    dev = torch.device("cuda", device)
    total, offs = 0, []
    for o in spec.objects:
        if o.kind == 0 and o.tier == TIER_DEVICE:
            total = _align(total, max(1, o.align))
            offs.append(total)
            total += o.size
        else:
            offs.append(None)
    if arena is None or arena.numel() < total:
        arena = torch.empty(max(total, 1), dtype=torch.uint8, device=dev)
    rs = RankState(spec.rank_id, spec.tp_idx, spec.pp_idx, spec.dp_idx, spec.seed, spec.metadata_bytes,
                   arena=arena)
    for o, off in zip(spec.objects, offs):
        so = StateObject(o.object_id, o.kind, o.tier if o.kind == 0 else TIER_HOST, o.precision, o.file_id,
                         o.size, o.space, o.offset)
        if o.kind == 0:
            # device-tier shards are views of the HBM arena; host-tier ones live
            # in pinned host memory (the pattern kernel writes them through UVA)
            so.payload = arena[off:off + o.size] if off is not None else \
                torch.empty(o.size, dtype=torch.uint8).pin_memory()
        so._meta = o.meta  # type: ignore[attr-defined]
        rs.objects.append(so)
    mutate_update_step(rs, iteration, stream)
    return rs


def pattern_descs(rank: RankState):
    raws = [o for o in rank.objects if o.is_raw()]
    arr = (N.PatternDesc * max(1, len(raws)))()
    for i, o in enumerate(raws):
        arr[i].data, arr[i].size, arr[i].space, arr[i].offset = (o.payload.data_ptr(), o.size_bytes,
                                                                 o.pattern_space, o.pattern_offset)
    return arr, len(raws)


def mutate_update_step(rank: RankState, iteration: int, stream=None):
    """mutate_update_step (model.cpp:233-244): every raw byte <- pattern(seed, space,
    iteration) by the pattern kernel; structured objects <- their value at
    `iteration` (metadata: make_metadata_value, tensor descriptors: iteration)."""
    arr, n = pattern_descs(rank)
    dev = rank.arena.device.index if rank.arena is not None else 0
    with torch.cuda.device(dev):
        sh = _stream_handle(stream)
    if n:
        N.call(N.lib.ts_pattern_fill, arr, n, rank.seed & (2**64 - 1), iteration, C.c_void_p(sh))
    for o in rank.objects:
        if o.is_raw():
            continue
        meta = getattr(o, "_meta", ("meta",))
        if meta[0] == "meta":
            o.structured = Value.metadata(rank.rank_id, rank.tp_idx, rank.pp_idx, rank.dp_idx, rank.seed,
                                          rank.metadata_bytes, iteration)
        else:
            _, name, dtype, numel, off, ln = meta
            o.structured = {"name": name, "dtype": dtype, "numel": numel, "shard_offset": off,
                            "shard_len": ln, "iteration": iteration}


def pattern_mismatches(rank: RankState, iteration: int, stream=None) -> int:
    """Bytes of the rank's raw objects that differ from pattern(iteration) (0 = bit-exact)."""
    arr, n = pattern_descs(rank)
    if not n:
        return 0
    dev = rank.arena.device.index if rank.arena is not None else 0
    with torch.cuda.device(dev):
        sh = _stream_handle(stream)
    out = C.c_uint64()
    N.call(N.lib.ts_pattern_verify, arr, n, rank.seed & (2**64 - 1), iteration, C.c_void_p(sh), C.byref(out))
    return out.value


# ---------------------------------------------------------------------------
# Restore / verify (format.cpp:430-529)


@dataclass
class VerifyReport:
    ok: bool
    files_checked: int
    objects_checked: int
    issues: List[tuple]


def file_cache_bytes() -> int:
    """Bytes of checkpoint-file pages currently page-locked for direct D2H."""
    return int(N.lib.ts_file_cache_bytes())


def file_cache_stats() -> Dict[str, int]:
    """Page-lock activity of the file registry since process start."""
    out = (C.c_uint64 * 5)()
    N.lib.ts_file_cache_stats(out)
    return {"registrations": out[0], "register_ns": out[1], "registered_bytes": out[2],
            "unregistrations": out[3], "unregister_ns": out[4]}


def file_cache_release_all() -> int:
    """Unlock every idle page-locked checkpoint file; returns the bytes released."""
    b = C.c_uint64(0)
    N.call(N.lib.ts_file_cache_release_all, C.byref(b))
    return int(b.value)


def retire_checkpoint(ckpt_dir: str, spare_dir: str):
    """Checkpoint rotation: invalidate `ckpt_dir` (manifest first) and move its files
    to `spare_dir` for reuse by engines with set_spare_dir(spare_dir)."""
    N.call(N.lib.ts_retire_checkpoint, ckpt_dir.encode(), spare_dir.encode())


def verify_checkpoint(manifest_path: str) -> VerifyReport:
    rep = N.VerifyReportC()
    cap = 4096
    iss = (N.VerifyIssue * cap)()
    N.call(N.lib.ts_verify, manifest_path.encode(), C.byref(rep), iss, cap)
    issues = [(N.FORMAT_KINDS.get(iss[i].kind, iss[i].kind), None if iss[i].object_id < 0 else iss[i].object_id)
              for i in range(min(rep.n_issues, cap))]
    return VerifyReport(bool(rep.ok), rep.files_checked, rep.objects_checked, issues)


class Restorer:
    """restore_checkpoint split per rank: open the manifest, list a rank's
    objects, restore it into caller-provided (or freshly allocated) shards."""

    def __init__(self, manifest_path: str, use_file_cache: bool = True, direct_io=None):
        """`use_file_cache`: read files this process page-locked (file_dma
        rotation) straight from their page cache; False: always pread.
        `direct_io`: True: other files' fixed regions are read O_DIRECT (disks);
        "uring": O_DIRECT through each reader thread's io_uring; False: pread;
        None (default): O_DIRECT only for files mostly absent from the page cache."""
        h = C.c_void_p()
        N.call(N.lib.ts_restore_open, manifest_path.encode(), C.byref(h))
        self.h = h.value
        self.last_stats: Dict[str, Any] = {}
        N.call(N.lib.ts_restore_set_file_cache, self.h, int(use_file_cache))
        dio = -1 if direct_io is None else 2 if direct_io == "uring" else int(bool(direct_io))
        N.call(N.lib.ts_restore_set_direct_io, self.h, dio)

    def __del__(self, _close=N.lib.ts_restore_close):
        h, self.h = getattr(self, "h", None), None
        if h:
            _close(h)

    def close(self):
        """Closes the handle; the last open one frees the restore staging
        (pinned ring + HBM window ring, up to ~4 GiB each)."""
        self.__del__()

    @property
    def n_ranks(self) -> int:
        return N.lib.ts_restore_n_ranks(self.h)

    def rank_info(self, index: int) -> N.RankInfo:
        ri = N.RankInfo()
        N.call(N.lib.ts_restore_rank_info, self.h, index, C.byref(ri))
        return ri

    def objects(self, index: int) -> List[N.RestoreObject]:
        n = C.c_size_t()
        N.call(N.lib.ts_restore_rank_objects, self.h, index, None, 0, C.byref(n))
        arr = (N.RestoreObject * max(1, n.value))()
        N.call(N.lib.ts_restore_rank_objects, self.h, index, arr, n.value, C.byref(n))
        return list(arr)[:n.value]

    def restore_rank(self, index: int, device: int = 0, into: Optional[RankState] = None,
                     stream=None) -> RankState:
        ri = self.rank_info(index)
        objs = self.objects(index)
        if into is None:
            total = sum(_align(o.size_bytes, 256) for o in objs if o.kind == 0)
            arena = torch.empty(max(total, 1), dtype=torch.uint8, device=torch.device("cuda", device))
            rs = RankState(ri.rank_id, ri.tp_idx, ri.pp_idx, ri.dp_idx, arena=arena)
            off = 0
            for o in objs:
                so = StateObject(o.object_id, o.kind, o.tier, o.precision, o.file_id, o.size_bytes)
                if o.kind == 0:
                    if o.tier == TIER_DEVICE:
                        so.payload = arena[off:off + o.size_bytes]
                        off += _align(o.size_bytes, 256)
                    else:
                        so.payload = torch.empty(o.size_bytes, dtype=torch.uint8).pin_memory()
                rs.objects.append(so)
        else:
            rs = into
        keep: list = []
        raws = RankState(rs.rank_id, objects=[o for o in rs.objects if o.is_raw()])
        arr = _desc_array(raws, keep)
        st = N.RestoreStats()
        with torch.cuda.device(device):
            sh = _stream_handle(stream)
        N.call(N.lib.ts_restore_rank, self.h, index, arr, len(raws.objects), device, C.c_void_p(sh), C.byref(st))
        self.last_stats = {f: getattr(st, f) for f, _ in N.RestoreStats._fields_}
        for o in rs.objects:
            if not o.is_raw():
                out = C.c_void_p()
                N.call(N.lib.ts_restore_structured, self.h, index, o.object_id, C.byref(out))
                o.structured = Value(out.value).to_py()
        return rs


def release_restore_staging() -> int:
    """Frees the process-wide restore staging now; returns the bytes freed."""
    return int(N.lib.ts_restore_release_staging())


def restore_checkpoint(manifest_path: str, device: int = 0, stream=None) -> List[RankState]:
    """restore_checkpoint (format.cpp:430-494): every rank's objects, raw payloads
    bit-identical on the GPU, structured values decoded, checksums verified."""
    r = Restorer(manifest_path)
    return [r.restore_rank(i, device, stream=stream) for i in range(r.n_ranks)]
