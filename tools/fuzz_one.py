import os, random, sys, tempfile
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
from test_gpu_fuzz import random_recipe, random_cfg
from gpu_helpers import checkpoint_recipe
seed = int(sys.argv[1])
rng = random.Random(1000 + seed)
rec = random_recipe(rng); cfg = random_cfg(rng)
print(cfg, [(len(r.objects), r.raw_bytes) for r in rec.ranks], flush=True)
with tempfile.TemporaryDirectory() as td:
    checkpoint_recipe(rec, td, cfg)
print("ok")
