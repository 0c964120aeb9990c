"""Multi-process manifest commit (world_size 2, gloo, CPU): each process
registers its own ranks; rank 0 commits a MANIFEST.tlv byte-identical to the
reference's for the same multi-rank checkpoint."""
import os
import socket
import sys

import pytest
import torch.multiprocessing as mp

from conftest import GOLDEN, ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, name, out_dir, result):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from paper_2601_16956_b200 import api, distributed as D
    from paper_2601_16956_b200 import synthetic as S

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    rec = S.load_recipe(os.path.join(GOLDEN, "recipes", name + ".recipe"))
    mine = [r for i, r in enumerate(rec.ranks) if i % ws == rank]
    sess = api.CheckpointSession(out_dir, rec.ckpt_id, rec.iteration, rec.manifest_echo(), n_ranks=len(rec.ranks),
                                 writes_manifest=rank == 0)
    for r in mine:
        sess.register_rank(api.RankState(r.rank_id, r.tp_idx, r.pp_idx, r.dp_idx, objects=[
            api.StateObject(o.object_id, o.kind, o.tier, o.precision, o.file_id, o.size) for o in r.objects]))
        sess.rank_persisted(r.rank_id)
    D.commit_manifest(sess, [r.rank_id for r in mine])
    base = D.global_object_id_base(sum(len(r.objects) for r in mine))
    result[rank] = base
    dist.destroy_process_group()


@pytest.mark.parametrize("name", ["tiny_layout", "two_ranks", "odd_layout"])
def test_manifest_commit_across_processes(tmp_path, name):
    ws = 2
    out = str(tmp_path / "ck")
    mgr = mp.Manager()
    result = mgr.dict()
    mp.start_processes(_worker, args=(ws, _free_port(), name, out, result), nprocs=ws, start_method="spawn")
    with open(os.path.join(out, "MANIFEST.tlv"), "rb") as f, \
            open(os.path.join(GOLDEN, "trees", name, "MANIFEST.tlv"), "rb") as g:
        assert f.read() == g.read()
    assert result[0] == 1 and result[1] > 1


def _gpu_worker(rank, ws, port, name, out_dir, result):
    """One OS process per rank, each with its own engine capturing its own
    shards on the GPU (both on cuda:0 on a 1-GPU box), files written
    independently, the manifest committed by rank 0 after the allgather."""
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    from paper_2601_16956_b200 import api, distributed as D
    from paper_2601_16956_b200 import synthetic as S

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    dev = rank % torch.cuda.device_count()
    torch.cuda.set_device(dev)
    rec = S.load_recipe(os.path.join(GOLDEN, "recipes", name + ".recipe"))
    mine = [r for i, r in enumerate(rec.ranks) if i % ws == rank]
    sess = api.CheckpointSession(out_dir, rec.ckpt_id, rec.iteration, rec.manifest_echo(), n_ranks=len(rec.ranks),
                                 writes_manifest=rank == 0)
    cfg = api.EngineConfig(staging_capacity_bytes=8 << 20, raw_chunk_bytes=1 << 20, flush_workers=2)
    tickets, engines = [], []
    for r in mine:
        st = api.materialize_payloads(r, dev, rec.pit)
        eng = api.CheckpointEngine(cfg, r.rank_id, dev)
        tickets.append((eng.issue_checkpoint(sess, st, rec.iteration), st))
        engines.append(eng)
    for t, _ in tickets:
        t.wait_persisted()
    D.commit_manifest(sess, [r.rank_id for r in mine])
    for e in engines:
        e.shutdown()
    result[rank] = [r.rank_id for r in mine]
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["two_ranks", "tiny_layout"])
def test_two_process_gpu_snapshot_tree_equals_reference(tmp_path, name):
    """engine.cpp:79-101 across OS processes: every file and MANIFEST.tlv of the
    tree equals the reference-written golden tree byte for byte."""
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from conftest import read_tree

    ws = 2
    out = str(tmp_path / "ck")
    mgr = mp.Manager()
    result = mgr.dict()
    mp.start_processes(_gpu_worker, args=(ws, _free_port(), name, out, result), nprocs=ws, start_method="spawn")
    assert sorted(result.keys()) == [0, 1]
    got, want = read_tree(out), read_tree(os.path.join(GOLDEN, "trees", name))
    assert sorted(got) == sorted(want)
    for k in want:
        assert got[k] == want[k], k
