"""Benchmark of the B200 snapshot path (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config cfg2] [--mode ring|direct|zerocopy]

Metric (BASELINE.json): checkpoint GB/s per GPU and per box, and training-blocked
ms per checkpoint. One step = one lazy checkpoint of this rank's state of the
named config (default cfg2: Llama-2 7B, ZeRO-1 over 8 ranks; rank r snapshots
shard r), i.e. update (pattern kernel rewrites every state byte) -> issue ->
snapshot complete (all bytes in pinned host memory) -> checksums complete.
Inputs (the state) live in HBM and are larger than L2. Multi-GPU: one process
per GPU, each snapshots its own shard (no data-path collective), value = all
ranks' bytes / max-over-ranks time.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import shutil
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# BASELINE.json's metric; `value` is the box GB/s, the blocked ms are in "blocked"
METRIC = "checkpoint GB/s per GPU & box (1/2/4/8 B200); training blocked ms/ckpt"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampler during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, device: int):
        self.samples = []
        self.dev = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), "--query-gpu=clocks.sm,clocks.max.sm,utilization.gpu,"
                 "clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap,power.draw", "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for s in self.samples for n, v in zip(names, s[4:8]) if v.lower() == "active"})
        pw = []
        for s in self.samples:
            try:
                pw.append(float(s[8]))
            except (IndexError, ValueError):
                pass
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples),
                "power_w": round(statistics.median(pw), 1) if pw else None}


def ncu_traffic(cfg: str, mode: str, pack_kernel: str, alg: float = 0.0):
    """DRAM bytes of the pack kernels of one checkpoint of this workload from
    the committed ncu capture (profiles/ncu_traffic.json: cfg2 full-shadow
    bulk+warp, cfg4 ring warp), else None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            t = json.load(f)
    except Exception:
        return None
    for e in t.get("entries", [t]):
        if e.get("workload") == cfg and mode == e.get("mode", "ring") and pack_kernel == e.get("pack_kernel", "warp"):
            if e.get("scale_with_alg") and alg:  # (captured with another ring size: same traffic per byte)
                return int(alg * e["traffic_bytes_per_launch"] / e["alg_bytes_per_launch"])
            return int(e["traffic_bytes_per_launch"])
    return None


def pcie_d2h_peak(dev) -> float:
    """Pinned D2H copy-engine rate of this GPU, measured in the same run (the
    D2H roofline): best of 3 x 2 GiB cudaMemcpyAsync into page-locked memory."""
    import torch

    n = 2 << 30
    src = torch.empty(n, dtype=torch.uint8, device=dev)
    dst = torch.empty(n, dtype=torch.uint8).pin_memory()
    best = 0.0
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dst.copy_(src, non_blocking=True)
        e1.record()
        e1.synchronize()
        best = max(best, n / (e0.elapsed_time(e1) / 1e3) / 1e9)
    del src, dst
    return best


def host_mem_avail() -> int:
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemAvailable:"):
                    return int(line.split()[1]) * 1024
    except Exception:
        pass
    return 0


def dist_info():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def workload_config(cfg: str, spec) -> dict:
    """The `config` object of both arms (ours and --impl reference): the named
    BASELINE.json workload; engine knobs go under "engine" in our line."""
    names = {"cfg1": "GPT-2 small generate_layout, 1 rank", "cfg1b": "GPT-2 small fp32 + Adam, 1 rank",
             "cfg2": "Llama-2 7B ZeRO-1 x8, rank-r shard", "cfg3": "Llama-2 13B ZeRO-3 x8, rank-r shard",
             "cfg4": "Llama-2 70B ZeRO-3 x8, rank-r shard (14 B/param)"}
    return {"workload": f"{cfg}: {names.get(cfg, cfg)}, {len(spec.objects)} objects, "
                        f"{spec.raw_bytes / 1e9:.3f} GB/rank",
            "l2": "inputs > L2 (126 MB)"}


def sample_recipe(cfg: str, rank: int, max_bytes: int):
    """Bounded sample of rank `rank`'s shard for the CPU reference: its raw
    objects in rank order until `max_bytes` (at least one; the whole rank when
    it fits), plus its metadata object. Same sizes and patterns as the full
    workload."""
    from paper_2601_16956_b200 import synthetic as S

    rec = S.config_recipe(cfg, rank)
    r = rec.ranks[0]
    raws, acc = [], 0
    for o in (o for o in r.objects if o.kind == 0):
        if raws and acc + o.size > max_bytes:
            break
        raws.append(o)
        acc += o.size
    whole = len(raws) == len([o for o in r.objects if o.kind == 0])
    metas = [o for o in r.objects if o.kind == 1 and (whole or o.meta[0] == "meta")]
    r.objects = [o for o in r.objects if (o.kind == 0 and o in raws) or o in metas]
    return rec, whole


REF_RATE_GUESS = 0.8e9  # B/s per reference process (FNV under its monitor; BASELINE.md §2, r1 box runs)


def run_reference(cfg: str, n: int, steps: int, warmup: int, budget_s: float):
    """The compiled reference (oracle/_ref/ts_ref_driver, built unmodified from
    /root/reference) as N independent OS processes, one per rank (BASELINE.md
    §3: never ranks as threads of one process), each pinned to its own disjoint
    set of host cores with its flush workers on all but one of them, each
    checkpointing a bounded sample of ITS rank's shard (`budget_s` of work for
    the whole run at the reference's rate), files on /dev/shm, one restore after
    the last step. Returns None when the driver is not built."""
    drv = os.path.join(ROOT, "oracle", "_ref", "ts_ref_driver")
    if not os.path.exists(drv):
        return None
    cores = sorted(os.sched_getaffinity(0))
    per = max(1, len(cores) // n)
    sets = [cores[i * per:(i + 1) * per] or cores[:1] for i in range(n)]
    reps = warmup + steps + 2  # (+ the restore, ~half the snapshot rate)
    want = int(budget_s / reps * REF_RATE_GUESS * (1.0 if per >= 4 else per / 4))
    avail = host_mem_avail()
    if avail:  # payload + staging cache + tmpfs files per process
        want = min(want, int(0.6 * avail / n / 3))
    tmp = tempfile.mkdtemp(dir="/dev/shm" if os.path.isdir("/dev/shm") else None)
    procs, meta = [], []
    try:
        for r in range(n):
            rec, whole = sample_recipe(cfg, r, want)
            b = rec.ranks[0].raw_bytes
            rp = os.path.join(tmp, f"rank{r}.recipe")
            with open(rp, "w") as f:
                f.write(rec.to_text())
            cap = 1 << (max(b, 256 << 20) - 1).bit_length()
            if avail and n * (2 * b + cap) > 0.8 * avail:
                cap = 256 << 20  # the reference's default cache (back-pressure)
            workers = max(1, len(sets[r]) - 1)
            cmd = ["taskset", "-c", ",".join(map(str, sets[r])), drv, "bench", rp, os.path.join(tmp, f"ckpt{r}"),
                   "--workers", str(workers), "--cache", str(cap), "--reps", str(steps), "--warmup", str(warmup),
                   "--restore-last"]
            if not shutil.which("taskset"):
                cmd = cmd[3:]
            procs.append(subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True))
            meta.append({"rank": r, "cores": sets[r], "workers": workers, "whole": whole,
                         "objects": len([o for o in rec.ranks[0].objects if o.kind == 0]), "cache": cap})
        outs = []
        for p in procs:
            out, err = p.communicate()
            if p.returncode != 0:
                raise RuntimeError(f"ts_ref_driver failed: {err.strip()[-500:]}")
            outs.append([json.loads(l) for l in out.splitlines() if l.startswith("{")])
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
        shutil.rmtree(tmp, ignore_errors=True)
    timed = [[x for x in rows if not x["warmup"]] for rows in outs]
    bytes_step = [t[0]["bytes"] for t in timed]
    snap = max(sum(x["snapshot_s"] for x in t) for t in timed)  # slowest rank (box metric)
    pers = max(sum(x["persist_s"] for x in t) for t in timed)
    rest = [x["restore_s"] for t in timed for x in t if x.get("restore_s", -1) > 0]
    k = len(timed[0])
    whole = all(m["whole"] for m in meta)
    return {"value": sum(bytes_step) * k / snap / 1e9, "persist_gbps": sum(bytes_step) * k / pers / 1e9,
            "steps": k, "ms_per_step": 1e3 * snap / k,
            "restore_gbps": round(sum(bytes_step) / max(rest) / 1e9, 4) if len(rest) == n else None,
            "bytes_per_step": int(sum(bytes_step)), "bytes_per_step_per_rank": bytes_step,
            "blocked_ms": 1e3 * max(statistics.mean(x["issue_s"] for x in t) for t in timed),
            "cores": sum(len(m["cores"]) for m in meta), "whole": whole,
            "sample": (f"{cfg}: {n} reference process(es), one per rank, each pinned to {per} core(s) "
                       f"({meta[0]['workers']} flush workers + 1 copier); per rank "
                       + ("the whole shard" if whole else
                          f"the first {meta[0]['objects']} raw objects of its shard + its metadata "
                          f"({bytes_step[0] / 1e9:.2f} GB of the {cfg} shard; the reference's rate is "
                          f"size-invariant, FNV-bound, BASELINE.md §2-3)")
                       + "; lazy, files on /dev/shm, restore once after the last step"),
            "procs": meta}


def reference_arm(args):
    """--impl reference: rank 0 alone (other torchrun ranks exit without work)
    runs one reference process per GPU of the run."""
    ws, rank, _ = dist_info()
    if rank != 0:
        return
    n = max(args.gpus, ws)
    r = run_reference(args.config, n, args.steps, args.warmup, args.ref_budget_s)
    if r is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/ts_ref_driver not built"}))
        return
    from paper_2601_16956_b200 import synthetic as S

    spec = S.config_recipe(args.config, 0).ranks[0]
    line = {"metric": METRIC, "impl": "reference", "value": round(r["value"], 4),
            "unit": "GB/s", "n_gpus": n, "steps": r["steps"], "warmup": args.warmup,
            "ms_per_step": round(r["ms_per_step"], 1), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": workload_config(args.config, spec),
            "sample": r["sample"], "bytes_per_step": r["bytes_per_step"],
            "persist_gbps": round(r["persist_gbps"], 4), "restore_gbps": r["restore_gbps"],
            "blocked_ms": round(r["blocked_ms"], 3),
            "cpu_baseline": {"value": round(r["value"], 4), "unit": "GB/s", "cores": r["cores"], "kind": "reference",
                             "sample": r["sample"]},
            "e2e": {"value": round(r["persist_gbps"], 4), "unit": "GB/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0,
                    "what": "issue -> files + footers + MANIFEST persisted (wait_persisted), /dev/shm"}}
    print(json.dumps(line))


def gemm_load(ms: float, dev, graph: bool = False, hbm_frac: float = 0.0):
    """Synthetic forward/backward for ~ms milliseconds: back-to-back bf16 GEMMs
    (compute-bound) interleaved, in 8 layer-like blocks, with an HBM-bound
    elementwise phase (bf16 a + b over 1 GiB operands: ~3 B of HBM traffic per
    element, the norm/activation/optimizer-style kernels of a real step) taking
    `hbm_frac` of the time; launched eagerly from Python or replayed as one
    CUDA graph."""
    import torch

    n = 8192
    a = torch.randn(n, n, device=dev, dtype=torch.bfloat16)
    b = torch.randn(n, n, device=dev, dtype=torch.bfloat16)
    c = torch.empty(n, n, device=dev, dtype=torch.bfloat16)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def per_call(fn):
        for _ in range(3):
            fn()
        e0.record()
        for _ in range(10):
            fn()
        e1.record()
        e1.synchronize()
        return e0.elapsed_time(e1) / 10

    gemm = lambda: torch.matmul(a, b, out=c)  # noqa: E731
    per_g = per_call(gemm)
    ew, per_e = None, 0.0
    if hbm_frac > 0:
        m = 1 << 29  # 512 Mi bf16 = 1 GiB per operand (>> L2)
        x = torch.randn(m, device=dev, dtype=torch.bfloat16)
        y = torch.randn(m, device=dev, dtype=torch.bfloat16)
        z = torch.empty(m, device=dev, dtype=torch.bfloat16)
        ew = lambda: torch.add(x, y, out=z)  # noqa: E731
        per_e = per_call(ew)
    blocks = 8
    reps_g = max(1, int(ms * (1 - hbm_frac) / per_g / blocks))
    reps_e = max(1, int(ms * hbm_frac / per_e / blocks)) if ew else 0

    def body():
        for _ in range(blocks):
            for _ in range(reps_g):
                gemm()
            for _ in range(reps_e):
                ew()

    total = blocks * (reps_g * per_g + reps_e * per_e)
    if graph:
        g = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            gemm()
            if ew:
                ew()
        torch.cuda.current_stream().wait_stream(side)
        with torch.cuda.graph(g):
            body()
        return g.replay, total
    return body, total


def ours(args):
    import torch
    import torch.distributed as dist

    from paper_2601_16956_b200 import api
    from paper_2601_16956_b200 import synthetic as S

    ws, rank, local = dist_info()
    # One GPU per rank (NCCL). TS_BENCH_SHARE_GPU=1 runs the N>1 path on fewer
    # GPUs than ranks (gloo, ranks share devices) — a functional check of the
    # multi-rank code path on a 1-GPU box, never a scaling number.
    local_ws = int(os.environ.get("LOCAL_WORLD_SIZE", str(ws)))
    share = os.environ.get("TS_BENCH_SHARE_GPU") == "1" or torch.cuda.device_count() < local_ws
    share_gpu = share
    local_dev = local % torch.cuda.device_count() if share else local
    backend = "gloo" if share else "nccl"
    if ws > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local_dev)
    dev = torch.device("cuda", local_dev)
    cdev = torch.device("cpu") if backend == "gloo" else dev  # collective tensors

    rec = S.config_recipe(args.config, rank)
    spec = rec.ranks[0]
    pcie_peak = pcie_d2h_peak(dev)
    state = api.materialize_payloads(spec, local_dev, 0)
    raw = spec.raw_bytes
    # D2H load balancing: a rank above the mean shard hands part
    # of its image to the copy engines of the GPUs below it (NVLink read, their
    # PCIe links). One allgather of shard sizes at setup; nothing per step.
    helpers, share = (), 0.0
    if ws > 1 and args.balance:
        sizes = [None] * ws
        dist.all_gather_object(sizes, (rank, local_dev, raw))
        mean = sum(s[2] for s in sizes) / ws
        if raw > 1.05 * mean:
            helpers = tuple(sorted({d for _, d, r in sizes if r < mean}))
            share = (raw - mean) / raw if helpers else 0.0
    img_est = raw + 4096 * (len(spec.objects) + 4)
    free, _ = torch.cuda.mem_get_info(local_dev)
    shadow = img_est + (256 << 20) <= free - (24 << 30)  # keep room for the GEMM load
    # no full shadow: the largest ring that leaves the same room (--ring-gb overrides)
    ring_bytes = int(args.ring_gb * (1 << 30)) if args.ring_gb else max(8 << 30, free - (26 << 30))
    # pinned pool: the whole image when host RAM allows (one pinning at engine
    # creation), else a bounded pool with back-pressure (staging.cpp semantics)
    local_ws = int(os.environ.get("LOCAL_WORLD_SIZE", str(ws)))
    avail = host_mem_avail()
    # Pinned pool: windows are released as they land (device checksums) or
    # once flushed / hashed; recycled files take the D2H directly (file_dma),
    # so a few GiB keep the copy engines busy (8 ranks x 4 GiB per node, not
    # 8 x the shard).
    pool_cap = int(args.pool_gb * (1 << 30)) if args.pool_gb else 4 << 30
    if avail:  # every rank of this node pins its pool: stay well inside host RAM
        pool_cap = min(pool_cap, max(1 << 30, int(0.3 * avail / max(1, local_ws))))
    pool = (min(img_est + (64 << 20), pool_cap) + (2 << 20) - 1) // (2 << 20) * (2 << 20)
    cfg = api.EngineConfig(d2h_mode=args.mode, staging_capacity_bytes=pool, raw_chunk_bytes=args.window_mb << 20,
                           device_staging_bytes=img_est + (1 << 20) if shadow else ring_bytes,
                           flush_workers=args.flush_workers or min(16, os.cpu_count() or 8), write_files=False,
                           checksum_on_gpu=not args.host_checksum, pack_kernel=args.pack_kernel,
                           checksum_priority=args.ck_priority, pack_priority=args.pack_priority,
                           checksum_host_frac=args.ck_host_frac, ring_chunk_bytes=int(args.ring_chunk_gb * (1 << 30)),
                           worker_nice=args.worker_nice, helper_devices=helpers, helper_share=share,
                           checksum_lane_max_bytes=-1 if args.lane_max_mb < 0 else int(args.lane_max_mb * (1 << 20)),
                           flush_mmap=3 if args.flush_uring else 2 if args.flush_direct else int(not args.flush_pwrite))
    eng = api.CheckpointEngine(cfg, spec.rank_id, local_dev)
    numa_node = eng.numa_node
    full = getattr(rec, "full_layout", None)
    echo = S.Recipe(layout=full).manifest_echo() if full else rec.manifest_echo()
    root = args.ckpt_root or ("/dev/shm" if os.path.isdir("/dev/shm") else tempfile.gettempdir())
    tdir = os.path.join(root, "ts_bench")
    if rank == 0:
        shutil.rmtree(tdir, ignore_errors=True)
        os.makedirs(tdir, exist_ok=True)
    if ws > 1:
        dist.barrier()
    launches0 = api.N.lib.ts_kernel_launch_count()

    def step(it, engine, write):
        api.mutate_update_step(state, it)
        sess = api.CheckpointSession(os.path.join(tdir, f"ckpt_{it:06d}") if write else "", it, it, echo,
                                     ws if write else 1, writes_manifest=write and rank == 0)
        t = engine.issue_checkpoint(sess, state, it)
        t.wait_snapshot()
        t.wait_persisted()
        if write:
            if ws > 1:  # the only collective: allgather of manifest blobs, rank 0 commits
                from paper_2601_16956_b200 import distributed as D
                D.commit_manifest(sess, [spec.rank_id])
            else:
                sess.wait_complete(600)
        st = t.stats()
        return st, sess

    it = 0
    for _ in range(args.warmup):
        it += 1
        step(it, eng, False)
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    stats = []
    l0 = api.N.lib.ts_kernel_launch_count()
    with Clocks(local_dev) as clk:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            it += 1
            st, _ = step(it, eng, False)
            stats.append(st)
        e1.record()
        torch.cuda.synchronize()
    launches = api.N.lib.ts_kernel_launch_count() - l0
    t_ms = e0.elapsed_time(e1)
    if ws > 1:
        tt = torch.tensor([t_ms], device=cdev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_ms = float(tt.item())
    bytes_step = stats[0]["total_bytes"]
    tot = torch.tensor([float(bytes_step)], device=cdev)
    if ws > 1:
        dist.all_reduce(tot)
    box_bytes = float(tot.item())
    value = box_bytes * args.steps / (t_ms / 1e3) / 1e9
    snap_ms = [s["t_snapshot_ns"] / 1e6 for s in stats]
    pack_ms = [s["pack_ms"] for s in stats]
    d2h_ms = [s["d2h_ms"] for s in stats]
    image = stats[0]["image_bytes"]
    hbm_peak, peak_kind = peaks()
    pack_alg = raw + image  # read every raw byte, write the image (incl. alignment gaps)
    packed = statistics.mean(s["packed_bytes"] for s in stats)
    if 0 < packed < image:  # HYBRID: the pack kernels handle the last ring-full only
        pack_alg = pack_alg * packed / image
    pack_mean = statistics.mean(pack_ms)
    # restore (one, after the loop): files written by the e2e phase below
    # --- e2e through the public API with files on /dev/shm -------------------
    e2e = None
    if args.e2e_steps > 0:
        # files kept on tmpfs: the retention window + the checkpoint in flight, per rank of the node
        try:
            st_shm = os.statvfs(os.path.dirname(tdir))
            shm_free = st_shm.f_bavail * st_shm.f_frsize
        except OSError:
            shm_free = 0
        # (rotation recycles the retired files: at most `keep` checkpoints exist at once)
        need = max(1, args.keep) * img_est * local_ws
        fits = not (shm_free and need > 0.85 * shm_free)
        if ws > 1:  # the same decision on every rank (the e2e phase has collectives)
            ft = torch.tensor([1 if fits else 0], device=cdev)
            dist.all_reduce(ft, op=dist.ReduceOp.MIN)
            fits = bool(ft.item())
        if not fits:
            print(f"bench: e2e skipped, needs ~{need / 1e9:.0f} GB of {shm_free / 1e9:.0f} GB tmpfs per node "
                  f"(use --keep 1)", file=sys.stderr)
            args.e2e_steps = 0
    if args.e2e_steps > 0:
        io_kw = {"write_files": True}
        if not os.path.realpath(root).startswith("/dev/shm") and not args.pool_gb:
            # a disk filesystem takes no file_dma: windows wait in the pool for
            # the (slower) page-cache flush, so give it the whole image when RAM allows
            io_kw["staging_capacity_bytes"] = (min(img_est + (64 << 20), max(pool, int(0.3 * avail / max(1, local_ws)))
                                               if avail else pool) + (2 << 20) - 1) // (2 << 20) * (2 << 20)
        cfg_io = api.EngineConfig(**{**cfg.__dict__, **io_kw})
        eng.shutdown()
        eng_io = api.CheckpointEngine(cfg_io, spec.rank_id, local_dev)
        spare = os.path.join(tdir, ".spare")
        if not args.fresh_files:
            eng_io.set_spare_dir(spare)
        # warm the file path: with rotation, 2 checkpoints fill the retention
        # window (fresh files, pool + flush; their pages get locked in the
        # background) and 2 more recycle them — the steady state is reached
        nwarm = 2 if args.fresh_files else 2 * args.keep
        for w in range(nwarm):
            it += 1
            old = os.path.join(tdir, f"ckpt_{it - args.keep:06d}")
            if not args.fresh_files and w >= args.keep and rank == 0 and os.path.exists(old):
                api.retire_checkpoint(old, spare)
            if ws > 1:
                dist.barrier()
            step(it, eng_io, True)
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record()
        dma, dio = [], []
        for _ in range(args.e2e_steps):
            it += 1
            # rotation: keep the last `keep` checkpoints, recycle older files
            old = os.path.join(tdir, f"ckpt_{it - args.keep:06d}")
            if not args.fresh_files and rank == 0 and os.path.exists(old):
                api.retire_checkpoint(old, spare)
            if ws > 1:
                dist.barrier()
            st, sess = step(it, eng_io, True)
            dma.append(st["file_dma_bytes"])
            dio.append(st["direct_io_bytes"])
        f1.record()
        torch.cuda.synchronize()
        e2e_ms = f0.elapsed_time(f1)
        if ws > 1:
            tt = torch.tensor([e2e_ms], device=cdev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e2e_ms = float(tt.item())
        e2e = {"value": round(box_bytes * args.e2e_steps / (e2e_ms / 1e3) / 1e9, 3), "unit": "GB/s",
               "persist_ms_last": round(st["t_persisted_ns"] / 1e6, 1),
               "snapshot_ms_last": round(st["t_snapshot_ns"] / 1e6, 1),
               "h2d_bytes_per_step": 0, "d2h_bytes_per_step": int(image),
               "file_dma_frac": round(sum(dma) / (len(dma) * image), 3) if dma else 0.0,
               "direct_io_frac": round(sum(dio) / (len(dio) * image), 3) if dio else 0.0,
               "what": f"issue -> files + footers + MANIFEST.tlv written to {root} (page cache), via the C-ABI"
                       + ("" if args.fresh_files else f"; rotation keeps {args.keep} checkpoint(s), older files recycled")
                       + ("; D2H windows land directly in the files' page-locked pages (file_dma)" if sum(dma) else
                          "; windows staged in the pinned pool, flushed by worker threads")}
        # restore of the last checkpoint (H2D + scatter-unpack + FNV verify)
        man = os.path.join(tdir, f"ckpt_{it:06d}", "MANIFEST.tlv")
        r = api.Restorer(man)
        ridx = [r.rank_info(i).rank_id for i in range(r.n_ranks)].index(spec.rank_id)
        free_now, _ = torch.cuda.mem_get_info(local_dev)
        if free_now > raw + (8 << 30):
            rs = r.restore_rank(ridx, local_dev)  # fresh shards (warms the file path)
            in_place = False
        else:  # no room for a second copy of the shard (cfg4): restore into the state itself
            rs, in_place = state, True
            r.restore_rank(ridx, local_dev, into=rs)  # warm-up (staging buffers), like the fresh case
        for o, so in zip(rs.objects, spec.objects):  # what pattern_mismatches checks against
            o.pattern_space, o.pattern_offset = so.space, so.offset
        rs.seed = spec.seed
        for o in rs.objects:  # zeroed destinations: a restore that skips bytes cannot pass
            if o.is_raw() and o.payload is not None:
                o.payload.zero_()
        torch.cuda.synchronize()
        # cold path (a restart: pread -> pinned -> H2D), then in-process
        # rollback (the files this process page-locked: H2D from the page cache)
        t0 = time.time()
        r2 = api.Restorer(man, use_file_cache=False)
        r2.restore_rank(ridx, local_dev, into=rs)
        torch.cuda.synchronize()
        restore_s = time.time() - t0
        bad_cold = api.pattern_mismatches(rs, it)
        for o in rs.objects:
            if o.is_raw() and o.payload is not None:
                o.payload.zero_()
        torch.cuda.synchronize()
        t0 = time.time()
        r3 = api.Restorer(man)
        r3.restore_rank(ridx, local_dev, into=rs)
        torch.cuda.synchronize()
        restore_warm_s = time.time() - t0
        for o, so in zip(rs.objects, spec.objects):
            o.pattern_space, o.pattern_offset = so.space, so.offset
        rs.seed = spec.seed
        bad = api.pattern_mismatches(rs, it)
        e2e["restore_gbps"] = round(raw / restore_s / 1e9, 3)
        e2e["restore_what"] = ("restore_gbps: files in the page cache but not page-locked by this process "
                               "(a restart: pread -> pinned ring -> H2D -> unpack; bound by the host's copy "
                               "bandwidth); restore_warm_gbps: files this process page-locked through "
                               "rotation (H2D straight from the page cache)")
        e2e["restore_warm_gbps"] = round(raw / restore_warm_s / 1e9, 3)
        e2e["restore_warm_direct_bytes"] = int(r3.last_stats.get("direct_bytes", 0))
        e2e["restore_bit_exact"] = bad == 0 and bad_cold == 0
        e2e["restore_into"] = "the live state (zeroed first)" if in_place else "fresh, zeroed shards"
        e2e["restore_stats"] = {k: (round(v, 4) if isinstance(v, float) else v) for k, v in r2.last_stats.items()}
        um = r2.last_stats.get("unpack_ms", 0.0)
        if um > 0:  # scatter-unpack kernel: reads the staged image, writes the shards (HBM roofline)
            ub = 2 * raw
            e2e["unpack_roofline"] = {"kernel": "unpack_kernel", "bound": "hbm", "achieved": round(ub / (um / 1e3) / 1e9, 1),
                                      "peak": hbm_peak, "unit": "GB/s", "frac": round(ub / (um / 1e3) / 1e9 / hbm_peak, 3),
                                      "alg_bytes": int(ub), "kernel_ms": round(um, 3)}
        del rs, r, r2, r3
        eng_io.shutdown()
    else:
        eng.shutdown()
    if ws > 1:
        dist.barrier()
    if rank == 0:
        shutil.rmtree(tdir, ignore_errors=True)
    if ws > 1:
        dist.barrier()
    api.file_cache_release_all()  # unlock the deleted checkpoints' pages

    # --- training-blocked time with a synthetic fwd/bwd load ------------------
    blocked = None
    if args.train_steps > 0:
        blocked = training_phase(args, api, state, spec, cfg, local_dev, dev, it, statistics.mean(snap_ms))

    # the TMA bulk kernel runs only for a full device shadow (engine.cpp run_job);
    # a multi-slot HBM ring (cfg4) packs every chunk with the warp kernel
    pack_used = "bulk" if ((shadow and args.pack_kernel != "warp") or args.pack_kernel == "bulk-ring") else "warp"
    pack_label = ("copy-engine DMA" if args.mode == "direct" else
                  "pack_bulk_kernel (TMA) + pack_kernel" if pack_used == "bulk" else
                  "pack_kernel (warp gather; last ring-full only, the head leaves by copy-engine DMA)"
                  if args.mode == "hybrid" else "pack_kernel (warp gather)")
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:  # (N=1 only)
        r = run_reference(args.config, 1, 3, 1, args.cpu_budget_s)
        if r:
            cpu = {"value": round(r["value"], 4), "unit": "GB/s", "cores": r["cores"], "kind": "reference",
                   "persist_gbps": round(r["persist_gbps"], 4), "restore_gbps": r["restore_gbps"],
                   "bytes_per_step": r["bytes_per_step"], "sample": r["sample"]}
    clocks = clk.summary()
    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "GB/s",
            "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(t_ms / args.steps, 2), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": workload_config(args.config, spec),
            "bytes_per_step": int(box_bytes),
            "engine": {"d2h_mode": args.mode, "device_shadow": bool(shadow),
                       "ring_gb": None if shadow else round(ring_bytes / 2**30, 1),
                       "pinned_pool_gb": round(pool / 2**30, 2),
                       "checksums": "host" if args.host_checksum else "gpu", "pack_kernel": args.pack_kernel,
                       "priorities": {"pack": args.pack_priority, "checksums": args.ck_priority},
                       "checksum_host_frac": "auto" if args.ck_host_frac < 0 else args.ck_host_frac,
                       "checksum_lane_max": ("auto" if args.lane_max_mb < 0 else
                                             f"{args.lane_max_mb} MiB" if args.lane_max_mb > 0 else "off"),
                       "lane_checksum_frac": round(statistics.mean(s["lane_checksum_bytes"] for s in stats)
                                                   / max(1, bytes_step), 3),
                       "lane_ms": round(statistics.mean(s["lane_ms"] for s in stats), 1),
                       "numa_node": numa_node, "shared_gpu": share_gpu,
                       "d2h_helpers": {"devices": list(helpers), "share": round(share, 3)},
                       "step": "update(pattern kernel) + issue + snapshot + checksums (no files)"},
            "per_gpu_gbps": round(value / ws, 3),
            "snapshot_ms_mean": round(statistics.mean(snap_ms), 2),
            "snapshot_gbps_mean": round(bytes_step / (statistics.mean(snap_ms) / 1e3) / 1e9, 3),
            "d2h_gbps": round(image / (statistics.mean(d2h_ms) / 1e3) / 1e9, 3) if min(d2h_ms) > 0 else None,
            "d2h_frac_pcie": round(image / (statistics.mean(d2h_ms) / 1e3) / 1e9 / pcie_peak, 3)
            if min(d2h_ms) > 0 else None,
            "pcie_d2h_peak_gbps": round(pcie_peak, 2),
            "roofline": {"kernel": pack_label,
                         "bound": "hbm", "achieved": round(pack_alg / (pack_mean / 1e3) / 1e9, 1),
                         "peak": hbm_peak, "peak_kind": peak_kind, "unit": "GB/s",
                         "frac": round(pack_alg / (pack_mean / 1e3) / 1e9 / hbm_peak, 3),
                         "traffic": ncu_traffic(args.config, args.mode, pack_used, pack_alg),
                         "traffic_source": "profiles/ncu_traffic.json (ncu --set full, same workload)",
                         "alg_bytes_per_launch": int(pack_alg),
                         "launch_ms": round(pack_mean, 3)},
            "gpu_launches": int(launches),
            "e2e": e2e, "blocked": blocked, "cpu_baseline": cpu, "clocks": clocks,
        }
        print(json.dumps(line))
    if ws > 1:
        dist.destroy_process_group()


def auto_interval(snapshot_ms: float, step_ms: float) -> int:
    """The most frequent checkpoint cadence (in steps) the D2H link sustains:
    one snapshot, with 10 % margin, must fit into the steps between two
    checkpoints."""
    return max(1, math.ceil(1.1 * snapshot_ms / max(step_ms, 1e-9)))


def training_phase(args, api, state, spec, cfg, local, dev, it0, snap_ms):
    """fwd+bwd (bf16 GEMMs) -> pre_update_barrier -> update -> issue, with and
    without checkpointing; reports host-blocked ms per checkpoint (issue_block +
    barrier_block, simulator.cpp:211-212) and the step-time slowdown."""
    import torch

    run, fb_ms = gemm_load(args.fwd_bwd_ms, dev, graph=args.fwd_bwd == "graph", hbm_frac=args.hbm_frac)
    # Checkpoint cadence: --ckpt-interval, or (0, default) the most frequent one
    # the D2H link sustains: a snapshot (measured above) must fit, with 10 %
    # margin, into the steps between two checkpoints. A 120.7 GB shard over one
    # PCIe Gen5 x16 link takes ~2.2 s, longer than a 1.8 s step: every 2 steps.
    interval = args.ckpt_interval or auto_interval(snap_ms, fb_ms)
    n_steps = -(-args.train_steps // interval) * interval  # whole checkpoint cycles per timed block
    # Long-lived objects (thousands of state descriptors) out of the cyclic GC's
    # reach, as training loops do: a full collection over them landed inside
    # random issue calls (up to ~270 ms for cfg4's 3,616 objects).
    import gc

    gc.collect()
    gc.freeze()
    # Checkpoints go where a deployment puts them: files on tmpfs with rotation
    # (keep `--keep`, file_dma), when tmpfs has room; else snapshot-only.
    ws, rank, _ = dist_info()
    local_ws = int(os.environ.get("LOCAL_WORLD_SIZE", str(ws)))
    tdir = os.path.join("/dev/shm", f"ts_train_r{rank}")
    files = False
    if args.train_files and os.path.isdir("/dev/shm"):
        st = os.statvfs("/dev/shm")
        files = max(1, args.keep) * spec.raw_bytes * 1.01 * local_ws < 0.85 * st.f_bavail * st.f_frsize
    if files:
        shutil.rmtree(tdir, ignore_errors=True)
        os.makedirs(tdir)
        cfg = api.EngineConfig(**{**cfg.__dict__, "write_files": True})
    # comparison strategies (engine.cpp:575-613): lazy (default), DataStates-Old
    # (lazy, structured objects serialized inline at issue), two_phase, sync
    strat = {"lazy": ("lazy", True), "lazy_old": ("lazy", False), "two_phase": ("two_phase", True),
             "sync": ("sync", True)}[args.strategy]
    cfg = api.EngineConfig(**{**cfg.__dict__, "strategy": strat[0], "lazy_serialize_overlap": strat[1]})
    eng = api.CheckpointEngine(cfg, spec.rank_id, local)
    spare = os.path.join(tdir, ".spare")
    if files:
        eng.set_spare_dir(spare)
    ckpts = []  # (dir, session, ticket) on disk, oldest first
    comp = torch.cuda.current_stream()
    res = {"off": ([], []), "lazy": ([], [])}
    host_ck, lane_ck, ck_tickets = [], [], []
    page_lock = {}  # file-registry page-lock activity inside the timed blocks (holds the driver)
    issue_cpp, issue_py = [], []  # issue time inside the engine vs the whole Python call
    clk = {"off": [], "lazy": []}
    fb_gpu = {"off": [], "lazy": []}  # CUDA-event time of fwd+bwd on the compute stream
    phases = {"off": [], "lazy": []}  # host wall per step phase
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    rot_wait = []
    it = it0

    def rotate_and_issue(it):
        tw = time.perf_counter()
        while len(ckpts) >= max(1, args.keep):  # rotation (a deployment does this off-thread)
            d0, _, t0k = ckpts.pop(0)
            t0k.wait_persisted()
            api.retire_checkpoint(d0, spare)
        rot_wait.append(time.perf_counter() - tw)
        d = os.path.join(tdir, f"ckpt_{it:06d}")
        sess = api.CheckpointSession(d, it, it, None, 1, writes_manifest=True)
        return d, sess

    if files:  # steady state first: the rotation window filled, recycled files page-locked
        for _ in range(2 * max(1, args.keep)):
            it += 1
            api.mutate_update_step(state, it, stream=comp)
            d, sess = rotate_and_issue(it)
            tk = eng.issue_checkpoint(sess, state, it, producer_stream=comp)
            ckpts.append((d, sess, tk))
            tk.wait_persisted()
        want = sum(max(0, (o.size + 4095) // 4096 * 4096) for o in spec.objects if o.kind == 0) * 0.9
        t_end = time.time() + 120
        while api.file_cache_bytes() < want * min(max(1, args.keep), len(ckpts)) and time.time() < t_end:
            time.sleep(0.2)
        rot_wait.clear()
    # off/lazy blocks alternate (twice) so clock / power-cap drift hits both arms
    for mode in ("off", "lazy", "off", "lazy"):
        pending = None
        times, blocked = res[mode]
        sampler = Clocks(local)
        sampler.__enter__()
        fc0 = api.file_cache_stats()
        for k in range(n_steps + 1):
            comp.synchronize()  # like a per-step loss.item(): the compute stream only, never the device
            t0 = time.perf_counter()
            ev0.record(comp)
            t_rec = time.perf_counter()
            run()                                    # forward + backward
            ev1.record(comp)
            t_launch = time.perf_counter()
            comp.synchronize()  # fwd/bwd done (the simulator's synchronous phases, simulator.cpp:129-130)
            if k > 0:
                fb_gpu[mode].append(ev0.elapsed_time(ev1))
            p_fb = time.perf_counter()
            b = eng.pre_update_barrier(pending, stream=comp, host_block=1) if pending else 0
            p_bar = time.perf_counter()
            it += 1
            api.mutate_update_step(state, it, stream=comp)  # optimizer update
            p_upd = time.perf_counter()
            ib = 0
            if mode == "lazy" and k % interval == 0:
                if files:
                    d, sess = rotate_and_issue(it)
                else:
                    sess = api.CheckpointSession("", it, it, None, 1, writes_manifest=False)
                tt = time.perf_counter()
                pending = eng.issue_checkpoint(sess, state, it, producer_stream=comp)
                ib = time.perf_counter() - tt
                if files:
                    ckpts.append((d, sess, pending))
                if k > 0:
                    st_k = pending.stats()
                    ck_tickets.append(pending)  # (checksum placement is known once prepared: read at the end)
                    issue_cpp.append(st_k["issue_block_ns"] / 1e6)
                    issue_py.append(1e3 * ib)
            p_iss = time.perf_counter()
            comp.synchronize()
            if k > 0:
                p_end = time.perf_counter()
                times.append(p_end - t0)
                phases[mode].append((p_fb - t0, t_rec - t0, t_launch - t_rec, p_bar - p_fb, p_upd - p_bar,
                                     p_iss - p_upd, p_end - p_iss))
                if mode == "lazy" and k % interval == 0:
                    blocked.append(1e3 * (b / 1e9 + ib))
                elif b and blocked:
                    blocked[-1] += 1e3 * b / 1e9  # barrier wait attributed to its checkpoint
        sampler.__exit__()
        clk[mode].append(sampler.summary())
        fc1 = api.file_cache_stats()
        pl = page_lock.setdefault(mode, {"registrations": 0, "register_ms": 0.0, "unregistrations": 0,
                                         "unregister_ms": 0.0})
        pl["registrations"] += fc1["registrations"] - fc0["registrations"]
        pl["register_ms"] += (fc1["register_ns"] - fc0["register_ns"]) / 1e6
        pl["unregistrations"] += fc1["unregistrations"] - fc0["unregistrations"]
        pl["unregister_ms"] += (fc1["unregister_ns"] - fc0["unregister_ns"]) / 1e6
        if pending:
            pending.wait_persisted()
        for tk in ck_tickets:
            tk.wait_persisted()
            host_ck.append(tk.stats()["host_checksum_bytes"] / max(1, spec.raw_bytes))
            lane_ck.append(tk.stats()["lane_checksum_bytes"] / max(1, spec.raw_bytes))
        ck_tickets.clear()
    res = {m: (statistics.mean(t), statistics.mean(b) if b else 0.0) for m, (t, b) in res.items()}
    eng.shutdown()
    dma = [t.stats()["file_dma_bytes"] for _, _, t in ckpts]
    ckpts.clear()
    if files:
        shutil.rmtree(tdir, ignore_errors=True)
        api.file_cache_release_all()
    off, lazy = res["off"][0], res["lazy"][0]
    return {"fwd_bwd_ms": round(fb_ms, 1), "fwd_bwd_launch": args.fwd_bwd, "steps": 2 * n_steps,
            "ckpt_interval": interval,
            "ckpt_interval_rule": ("--ckpt-interval" if args.ckpt_interval else
                                   f"auto: ceil(1.1 x snapshot {snap_ms:.0f} ms / fwd+bwd {fb_ms:.0f} ms)"),
            "hbm_bound_frac": args.hbm_frac, "strategy": args.strategy,
            "step_ms_no_ckpt": round(1e3 * off, 2), "step_ms_lazy_ckpt": round(1e3 * lazy, 2),
            "slowdown_pct": round(100 * (lazy - off) / off, 2),
            "blocked_ms_per_ckpt": round(res["lazy"][1], 3),
            "host_checksum_frac": round(statistics.mean(host_ck), 3) if host_ck else None,
            "lane_checksum_frac": round(statistics.mean(lane_ck), 3) if lane_ck else None,
            "rotation_wait_ms": round(1e3 * statistics.mean(rot_wait), 2) if rot_wait else None,
            "issue_ms": {"engine": round(statistics.mean(issue_cpp), 3) if issue_cpp else None,
                         "python_call": round(statistics.mean(issue_py), 3) if issue_py else None},
            "fwd_bwd_gpu_ms": {m: round(statistics.mean(v), 1) for m, v in fb_gpu.items() if v},
            "phase_ms": {m: dict(zip(["fwd_bwd", "fwd_bwd_event_record", "fwd_bwd_launch", "barrier", "update_launch",
                                      "issue", "final_sync"],
                                     [round(1e3 * statistics.mean(x), 2) for x in zip(*v)]))
                         for m, v in phases.items() if v},
            "phase_ms_max": {m: dict(zip(["fwd_bwd", "fwd_bwd_event_record", "fwd_bwd_launch", "barrier",
                                          "update_launch", "issue", "final_sync"],
                                         [round(1e3 * max(x), 2) for x in zip(*v)]))
                             for m, v in phases.items() if v},
            "fwd_bwd_gpu_ms_max": {m: round(max(v), 1) for m, v in fb_gpu.items() if v},
            "page_lock_in_blocks": {m: {k: round(v, 1) for k, v in d.items()} for m, d in page_lock.items()},
            "fwd_bwd_event_record_ms_per_step": {m: [round(1e3 * x[1], 2) for x in v] for m, v in phases.items() if v},
            "clocks": {m: {"sm_mhz": [c["sm_mhz"] for c in v], "power_w": [c.get("power_w") for c in v],
                           "reasons": sorted({r for c in v for r in c["reasons"]})} for m, v in clk.items()},
            "checkpoints_to": (f"files on /dev/shm, rotation keeps {args.keep}, file_dma bytes of the last "
                               f"{len(dma)}: {dma}") if files else "snapshot only (pinned pool)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg4",
                    help="BASELINE.json workload: cfg4 (70B ZeRO-3 shard, the north-star config, default), "
                         "cfg1, cfg1b, cfg2, cfg3")
    ap.add_argument("--mode", default="hybrid", choices=["ring", "direct", "zerocopy", "hybrid"])
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--train-steps", type=int, default=8,
                    help="timed steps per off/lazy block (rounded up to whole checkpoint cycles)")
    ap.add_argument("--fwd-bwd-ms", type=float, default=1800.0)
    ap.add_argument("--fwd-bwd", default="graph", choices=["graph", "eager"],
                    help="synthetic fwd/bwd launched as one CUDA graph (default) or eagerly from Python")
    ap.add_argument("--ckpt-interval", type=int, default=0,
                    help="checkpoint every k training steps (0 = auto: the most frequent cadence the D2H sustains)")
    ap.add_argument("--strategy", default="lazy", choices=["lazy", "lazy_old", "two_phase", "sync"],
                    help="training phase: checkpoint strategy (the reference's comparison arms)")
    ap.add_argument("--hbm-frac", type=float, default=0.35,
                    help="share of the synthetic fwd/bwd spent in an HBM-bound elementwise phase")
    ap.add_argument("--host-checksum", action="store_true", help="FNV on host threads instead of the GPU kernels")
    ap.add_argument("--pack-kernel", default="bulk", choices=["warp", "bulk", "bulk-ring"],
                    help="bulk: TMA cp.async.bulk for large 16-B aligned fragments + warp kernel for the rest")
    ap.add_argument("--ck-priority", type=int, default=-1, help="device checksum stream priority (1/0/-1)")
    ap.add_argument("--ck-host-frac", type=float, default=-1.0,
                    help="share of checksums on host workers (0: all GPU; <0: auto from host rate and cadence)")
    ap.add_argument("--pack-priority", type=int, default=1, help="capture (pack) stream priority (1/0/-1)")
    ap.add_argument("--lane-max-mb", type=float, default=0.0,
                    help="lane-serial device checksums for objects up to this size (0 off, -1 auto)")
    ap.add_argument("--flush-workers", type=int, default=0, help="host worker threads (default: min(16, cores))")
    ap.add_argument("--keep", type=int, default=1, help="e2e rotation: checkpoints kept on tmpfs")
    ap.add_argument("--ckpt-root", default="", help="e2e checkpoint directory root (default /dev/shm)")
    ap.add_argument("--flush-pwrite", action="store_true", help="pool flushes with pwrite(2) instead of mmap copies")
    ap.add_argument("--flush-direct", action="store_true",
                    help="pool flushes with O_DIRECT pwrite from the pinned windows (disk filesystems)")
    ap.add_argument("--flush-uring", action="store_true",
                    help="as --flush-direct, each window body submitted through io_uring (4 MiB writes in flight)")
    ap.add_argument("--window-mb", type=int, default=64, help="D2H window (raw_chunk_bytes) in MiB")
    ap.add_argument("--no-train-files", dest="train_files", action="store_false",
                    help="training phase: snapshot only (no files)")
    ap.add_argument("--fresh-files", action="store_true",
                    help="e2e: new files every checkpoint (no rotation / recycling)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget-s", type=float, default=30.0,
                    help="cpu_baseline: seconds of reference CPU work (bounded sample of the workload)")
    ap.add_argument("--ref-budget-s", type=float, default=200.0,
                    help="--impl reference: seconds of reference work for the whole --steps/--warmup run")
    ap.add_argument("--pool-gb", type=float, default=0.0, help="pinned pool cap (default 4 GiB)")
    ap.add_argument("--ring-gb", type=float, default=0.0,
                    help="HBM staging ring when no full device shadow fits (0 = auto: free HBM - 26 GiB)")
    ap.add_argument("--ring-chunk-gb", type=float, default=0.0, help="ring slot size (0 = auto)")
    ap.add_argument("--worker-nice", type=int, default=19, help="nice increment of engine worker threads")
    ap.add_argument("--no-balance", dest="balance", action="store_false",
                    help="N>1: no D2H load balancing onto helper GPUs")
    args = ap.parse_args()
    if args.impl == "reference":
        reference_arm(args)
        return
    ws = int(os.environ.get("WORLD_SIZE", "0"))
    if ws == 0 and args.gpus > 1:
        # one process per GPU: launch the ranks ourselves (same as the driver's
        # torchrun command), rank 0 prints the line
        import socket

        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    if ws and ws != args.gpus:
        sys.exit(f"bench: WORLD_SIZE={ws} but --gpus {args.gpus}")
    ours(args)


if __name__ == "__main__":
    main()
