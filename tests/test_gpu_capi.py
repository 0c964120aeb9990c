"""The C-ABI on its own (include/ts_b200.h): a C++ program with no Python or
torch in it (tests/capi/capi_checkpoint.cpp) checkpoints every rank of a golden
recipe through ts_issue, restores it bit-exactly and verifies it. The tree it
writes must equal the one the reference wrote."""
import json
import os
import subprocess

import pytest

from conftest import GOLDEN, ROOT, golden_recipes, read_tree
from paper_2601_16956_b200 import build as B
from paper_2601_16956_b200 import synthetic as S

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def driver(tmp_path_factory):
    lib = B.build()
    exe = str(tmp_path_factory.mktemp("capi") / "capi_checkpoint")
    subprocess.run(["g++", "-O2", "-std=c++17", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
                    os.path.join(ROOT, "tests", "capi", "capi_checkpoint.cpp"), "-o", exe,
                    "-L", os.path.dirname(lib), "-lts_b200", "-L", "/usr/local/cuda/lib64", "-lcudart_static",
                    "-ldl", "-lrt", "-lpthread", "-Wl,-rpath," + os.path.dirname(lib)], check=True)
    return exe


def spec_text(rec: S.Recipe) -> str:
    out = [f"checkpoint {rec.ckpt_id} {rec.iteration}", f"pattern_iteration {rec.pit}"]
    echo = rec.manifest_echo()
    if echo:
        out.append("echo {tp} {pp} {dp} {zero1} {seed} {n_params} {layers} {metadata_bytes}".format(**echo))
    for r in rec.ranks:
        out.append(f"rank {r.rank_id} {r.tp_idx} {r.pp_idx} {r.dp_idx} {r.seed} {r.metadata_bytes}")
        for o in r.objects:
            if o.kind == 0:
                out.append(f"raw {o.object_id} {o.file_id} {o.precision} {o.tier} {o.size} {o.space} {o.offset}")
            else:
                out.append(f"meta {o.object_id} {o.file_id}")
    return "\n".join(out) + "\n"


def eligible(name):
    rec = S.load_recipe(os.path.join(GOLDEN, "recipes", name + ".recipe"))
    ok = all((o.kind == 0 and o.tier == 0) or (o.kind == 1 and o.meta[0] == "meta")
             for r in rec.ranks for o in r.objects)
    return ok and sum(r.raw_bytes for r in rec.ranks) < (1 << 30)


@pytest.mark.parametrize("name", [n for n in golden_recipes() if eligible(n)])
def test_capi_only_checkpoint_equals_reference(gpu, driver, tmp_path, name):
    rec = S.load_recipe(os.path.join(GOLDEN, "recipes", name + ".recipe"))
    spec = tmp_path / "spec.txt"
    spec.write_text(spec_text(rec))
    out = tmp_path / "ckpt"
    r = subprocess.run([driver, str(spec), str(out)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr + r.stdout
    res = json.loads(r.stdout.strip().splitlines()[-1])
    assert res["restore_mismatched_bytes"] == 0 and res["verify_ok"] == 1
    assert read_tree(str(out)) == read_tree(os.path.join(GOLDEN, "trees", name))
