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
