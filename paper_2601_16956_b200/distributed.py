"""Multi-process (one process per GPU) plumbing around the engine.

The snapshot data path has no collective: every rank captures its own shard.
The only exchange is this module's allgather of per-rank manifest blobs
(object ids, files, kinds — the TLV manifest_rank_info of format.cpp:310-335)
so that global rank 0 can commit MANIFEST.tlv after every rank persisted
(manifest-last, engine.cpp:79-101), plus an exclusive scan for global object
ids when ranks build their states independently (model.cpp:108 numbers them
globally). NCCL over NVLink on GPU process groups, gloo on CPU ones.
"""
from __future__ import annotations

from typing import List, Sequence

import torch
import torch.distributed as dist


def _device_for(group=None) -> torch.device:
    backend = dist.get_backend(group)
    if backend == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def allgather_bytes(payload: bytes, group=None) -> List[bytes]:
    """Allgather of variable-length byte strings (length allgather + padded allgather)."""
    dev = _device_for(group)
    ws = dist.get_world_size(group)
    n = torch.tensor([len(payload)], dtype=torch.int64, device=dev)
    lens = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(ws)]
    dist.all_gather(lens, n, group=group)
    mx = max(int(x.item()) for x in lens)
    buf = torch.zeros(max(mx, 1), dtype=torch.uint8, device=dev)
    if payload:
        buf[:len(payload)] = torch.frombuffer(bytearray(payload), dtype=torch.uint8).to(dev)
    outs = [torch.zeros_like(buf) for _ in range(ws)]
    dist.all_gather(outs, buf, group=group)
    return [bytes(o[:int(l.item())].cpu().numpy().tobytes()) for o, l in zip(outs, lens)]


def _pack(blobs: Sequence[bytes]) -> bytes:
    out = bytearray(len(blobs).to_bytes(8, "little"))
    for b in blobs:
        out += len(b).to_bytes(8, "little") + b
    return bytes(out)


def _unpack(data: bytes) -> List[bytes]:
    n = int.from_bytes(data[:8], "little")
    pos, out = 8, []
    for _ in range(n):
        ln = int.from_bytes(data[pos:pos + 8], "little")
        out.append(data[pos + 8:pos + 8 + ln])
        pos += 8 + ln
    return out


def commit_manifest(session, local_rank_ids: Sequence[int], group=None, writer: int = 0,
                    timeout_s: float = 600.0) -> None:
    """Call on every process after its local ranks' tickets persisted. The
    writer process (whose session was created with writes_manifest=True) adds
    the remote ranks' info and writes MANIFEST.tlv; all processes return after
    the commit (a barrier), so the checkpoint is complete everywhere."""
    me = dist.get_rank(group)
    payload = _pack([session.rank_blob(r) for r in local_rank_ids])
    gathered = allgather_bytes(payload, group)
    if me == writer:
        for src, data in enumerate(gathered):
            if src == writer:
                continue
            for blob in _unpack(data):
                session.add_remote_rank(blob)
        session.wait_complete(timeout_s)
    dist.barrier(group)


def global_object_id_base(n_local_objects: int, group=None, first_id: int = 1) -> int:
    """Exclusive scan of per-rank object counts: the first global object id of
    this rank (ids are global across ranks, model.cpp:108)."""
    dev = _device_for(group)
    ws = dist.get_world_size(group)
    t = torch.tensor([n_local_objects], dtype=torch.int64, device=dev)
    outs = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(ws)]
    dist.all_gather(outs, t, group=group)
    me = dist.get_rank(group)
    return first_id + sum(int(o.item()) for o in outs[:me])
