"""Probe the GPU box: host RAM/cores/storage and pinned PCIe copy bandwidth."""
import json, os, subprocess, time
import torch

def sh(c):
    try:
        return subprocess.run(c, shell=True, capture_output=True, text=True, timeout=60).stdout
    except Exception as e:
        return str(e)

out = {}
out["nproc"] = os.cpu_count()
out["lscpu"] = sh("lscpu | head -30")
out["free"] = sh("free -g")
out["df"] = sh("df -h /dev/shm /tmp / 2>/dev/null")
out["smi"] = sh("nvidia-smi; nvidia-smi topo -m")
out["numa"] = sh("numactl -H 2>/dev/null || ls /sys/devices/system/node")
out["ulimit"] = sh("ulimit -a")
dev = torch.device("cuda:0")
res = {}
for gb in [1, 4, 16]:
    n = gb << 30
    t0 = time.time()
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    tpin = time.time() - t0
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    d.fill_(1)
    torch.cuda.synchronize()
    s = torch.cuda.Stream(priority=-1)
    for direction in ["d2h", "h2d"]:
        best = 0
        for i in range(4):
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(s):
                e0.record()
                if direction == "d2h":
                    h.copy_(d, non_blocking=True)
                else:
                    d.copy_(h, non_blocking=True)
                e1.record()
            e1.synchronize()
            ms = e0.elapsed_time(e1)
            best = max(best, n / ms / 1e6)
        res[f"{direction}_{gb}GiB_GBps"] = round(best, 2)
    res[f"pin_{gb}GiB_s"] = round(tpin, 3)
    # device copy
    d2 = torch.empty_like(d)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    d2.copy_(d); torch.cuda.synchronize()
    e0.record(); d2.copy_(d); e1.record(); e1.synchronize()
    res[f"d2d_{gb}GiB_GBps_rw"] = round(2 * n / e0.elapsed_time(e1) / 1e6, 1)
    del h, d, d2
    torch.cuda.empty_cache()
out["bw"] = res
# page-cache write speed to /dev/shm and /tmp
import numpy as np
buf = np.ones(1 << 30, dtype=np.uint8)
for p in ["/dev/shm/probe.bin", "/tmp/probe.bin"]:
    try:
        t0 = time.time()
        with open(p, "wb") as f:
            for _ in range(4):
                f.write(buf)
        out[f"write_{p}_GBps"] = round(4 / (time.time() - t0), 2)
        os.remove(p)
    except Exception as e:
        out[f"write_{p}"] = str(e)
print(json.dumps(out["bw"]))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/probe_box.json", "w"), indent=1)
