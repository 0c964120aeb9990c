"""GPU FNV throughput: 8 x 1 GiB objects + 20k x 64 KiB fragments."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
from paper_2601_16956_b200 import api
buf = torch.randint(0, 256, (8 << 30,), dtype=torch.uint8, device="cuda")
big = [buf[i << 30:(i + 1) << 30] for i in range(8)]
small = [buf[i * 65536:(i + 1) * 65536 - 7] for i in range(20000)]
for name, objs in (("8x1GiB", big), ("20k x 64KiB", small)):
    api.fnv1a64_device(objs)
    torch.cuda.synchronize(); t = time.time()
    for _ in range(3):
        api.fnv1a64_device(objs)
    torch.cuda.synchronize(); dt = (time.time() - t) / 3
    n = sum(o.numel() for o in objs)
    print(name, f"{n / dt / 1e9:.1f} GB/s", f"{1e3 * dt / (n / 1e9):.3f} ms/GB")
