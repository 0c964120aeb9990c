import os, sys, tempfile
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
from gpu_helpers import checkpoint_recipe, tree_bytes
from paper_2601_16956_b200 import api, synthetic as S
name, mode = sys.argv[1], sys.argv[2]
rec = S.load_recipe(f"tests/golden/recipes/{name}.recipe")
cfg = api.EngineConfig(d2h_mode=mode, raw_chunk_bytes=64 << 10, staging_capacity_bytes=1 << 20,
                       device_staging_bytes=256 << 10, flush_workers=3)
with tempfile.TemporaryDirectory() as td:
    checkpoint_recipe(rec, td, cfg)
    ok = tree_bytes(td) == tree_bytes(f"tests/golden/trees/{name}")
print(name, mode, "IDENTICAL" if ok else "DIFFERENT", flush=True)
