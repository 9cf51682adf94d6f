#!/usr/bin/env python3
"""bench.py -- Mcells/s of the B200 power-diagram path on BASELINE.json's headline workload.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl ours|reference]

A "step" is one full pd_build (pack, Morton, sort, LBVH, refit, cell kernel, CSR) over the whole
synthetic workload, inputs resident in HBM (value), and the same through the C ABI with pinned host
buffers + host outputs (e2e).  At N=1 the workload is C4 (10M scene-like power diagram,
BASELINE.json configs[3], the config the metric is quoted on).  For N>1 (torchrun, one rank per GPU)
the cells are split into Morton slices (strong scaling: the 10M diagram is fixed), exchanged with
NCCL inside libpd (pd_build_sharded: rank-0 input, LBVH broadcast, owner broadcasts of the slices, assembly
on every rank); time = max over ranks.

`--impl reference` times the CPU oracle (oracle/, the reference arm of this tier) on host cores on a
bounded sample of the same workload's cells per step; under torchrun only rank 0 runs it.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "Mcells/s for 10M-point power diagram"
UNIT = "Mcells/s"
# Algorithmic FP work per cell (SURVEY.md §8(d) "Algorithmic work per cell": W_min ≈ 25·300 node
# tests + 15·450 site tests + 4·27·77 vertex classifications + 40·27 vertex creations ≈ 2.3e4
# FP ops/cell).  The peak is MEASURED in the same job (pd_measure_fp32_peak); the nominal
# 148 SMs × 128 FP32 lanes × 1.965 GHz is reported beside it.
W_MIN_OPS_PER_CELL = 2.3e4
ALU_PEAK_TOPS = 148 * 128 * 1.965e9 / 1e12


def _env_rank():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


class ClockSampler:
    """nvidia-smi sampled every 200 ms during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.sw_power_cap,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def load_workload(cfg: str, n: int | None):
    import pdgen
    t = time.time()
    wl = pdgen.make(cfg, n=n)
    return wl, time.time() - t


def cpu_baseline(wl, budget_s: float = 15.0, seed: int = 7):
    """The oracle as it stands, on host cores, on a bounded random sample of the workload's cells."""
    import oracle
    threads = os.cpu_count() or 1
    rng = np.random.default_rng(seed)
    probe = rng.choice(wl.n, size=min(wl.n, 2 * threads), replace=False)
    t = time.time()
    oracle.cells(wl.points, wl.weights, wl.box, ids=probe, threads=threads)
    dt = max(time.time() - t, 1e-6)
    m = int(min(wl.n, max(len(probe), len(probe) * budget_s / dt)))
    ids = rng.choice(wl.n, size=m, replace=False)
    t = time.time()
    oracle.cells(wl.points, wl.weights, wl.box, ids=ids, threads=threads)
    dt = time.time() - t
    return {"value": m / dt / 1e6, "unit": UNIT, "cores": threads, "kind": "oracle",
            "sample": f"{m} random cells of {wl.name} ({wl.n} sites), full brute-force clip per cell, "
                      f"{dt:.1f} s wall on {threads} threads"}


def cpu_reference(wl, budget_s: float = 10.0, seed: int = 8):
    """the CPU reference of the same definition (oracle/pd_oracle.c orc_kd_*: the oracle's
    clipper fed by a best-first walk of a weight-augmented k-d tree, stopped by the weighted radius of
    security), all host threads, on a bounded random sample of the workload's cells.  The tree is built once
    (timed separately); `value` is cells / query time, `value_with_build` charges the build to the whole
    diagram (N / (build + N x per-cell time))."""
    import oracle
    threads = os.cpu_count() or 1
    t = time.time()
    kr = oracle.KdReference(wl.points, wl.weights, wl.box)
    build_s = time.time() - t
    rng = np.random.default_rng(seed)
    probe = rng.choice(wl.n, size=min(wl.n, 256 * threads), replace=False)
    t = time.time()
    kr.cells(probe, threads=threads)
    dt = max(time.time() - t, 1e-6)
    m = int(min(wl.n, max(len(probe), len(probe) * budget_s / dt)))
    ids = rng.choice(wl.n, size=m, replace=False)
    t = time.time()
    kr.cells(ids, threads=threads)
    dt = time.time() - t
    kr.close()
    v = m / dt / 1e6
    return {"value": v, "unit": UNIT, "cores": threads,
            "kind": "k-d tree (per-subtree max weight) + weighted radius of security, same definition",
            "build_s": round(build_s, 2), "value_with_build": wl.n / (build_s + wl.n / (v * 1e6)) / 1e6,
            "sample": f"{m} random cells of {wl.name} ({wl.n} sites), {dt:.1f} s wall on {threads} threads; "
                      f"tree build {build_s:.1f} s (single thread) reported apart"}


def profile_metrics():
    """ncu counters of the tier-1 cell kernel (C4, 10M sites) from this round's capture, committed under
    profiles/ by tools/profile_round.sh: DRAM bytes per launch (roofline.traffic), FP32 lane-ops, L2 bytes,
    issue / occupancy / divergence.  ncu cannot run inside the timed bench; the file names its capture."""
    for name in ("r2_cells_metrics.json", "cells_kernel_traffic.json"):
        p = os.path.join(ROOT, "profiles", name)
        if os.path.exists(p):
            try:
                d = json.load(open(p))
                d["_file"] = "profiles/" + name
                return d
            except Exception:
                pass
    return None


def run_reference(args):
    rank, world, _ = _env_rank()
    if world > 1 and rank != 0:
        return 0
    import oracle
    wl, _ = load_workload(args.config, args.n)
    threads = os.cpu_count() or 1
    per_step = max(threads, args.ref_cells)
    rng = np.random.default_rng(11)
    times = []
    for it in range(args.warmup + args.steps):
        ids = rng.choice(wl.n, size=per_step, replace=False)
        t = time.time()
        oracle.cells(wl.points, wl.weights, wl.box, ids=ids, threads=threads)
        dt = time.time() - t
        if it >= args.warmup:
            times.append(dt)
    ms = 1e3 * float(np.mean(times))
    value = per_step / (ms / 1e3) / 1e6
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": f"{wl.name}: {wl.description}", "n": wl.n,
                       "sample_per_step": per_step},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle",
                             "sample": f"{per_step} random cells of {wl.name} per step"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import torch
    import torch.distributed as dist
    import paper_2605_06408_b200 as pd
    from paper_2605_06408_b200 import build as pdbuild
    from paper_2605_06408_b200 import dist as pddist

    rank, world, local = _env_rank()
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    if rank == 0:
        pdbuild.build()
    if world > 1:
        dist.barrier()
    pd.load_library()
    dev = torch.device("cuda", local)
    # the workload lives on rank 0 (points start on rank 0); the others learn n
    wl, gen_s = (load_workload(args.config, args.n) if rank == 0 else (None, 0.0))
    n = wl.n if rank == 0 else 0
    if world > 1:
        obj = [n]
        dist.broadcast_object_list(obj, src=0)
        n = obj[0]
    p = torch.from_numpy(wl.points).to(dev) if rank == 0 else None
    w = (None if wl.weights is None else torch.from_numpy(wl.weights).to(dev)) if rank == 0 else None
    box = wl.box if rank == 0 else None
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # 256 MiB > 126 MB L2
    stream = torch.cuda.current_stream(dev)
    comm = pddist.init_comm(device=local) if world > 1 else None

    base_flags = pd.WARM_START if args.warm_start else (pd.WARM_ADAPTIVE if args.warm_adaptive else 0)

    def step(flags=0, host=False):
        flags |= base_flags
        pts, wts = (p, w) if not host else (hp.numpy() if rank == 0 else None,
                                           (None if hw is None else hw.numpy()) if rank == 0 else None)
        if world > 1:  # pd_build_sharded: rank-0 input, NCCL broadcast of the LBVH, slice, exchange, assemble
            return pd.build_sharded(comm, pts, wts, box, n=n, leaf_size=args.leaf, flags=flags, out_host=host)
        return pd.build_diagram(pts, wts, box, leaf_size=args.leaf, flags=flags, out_host=host)

    hp = torch.from_numpy(wl.points).pin_memory() if rank == 0 else None
    hw = (None if wl.weights is None else torch.from_numpy(wl.weights).pin_memory()) if rank == 0 else None
    for _ in range(args.warmup):
        d = step()
        del d
    torch.cuda.synchronize()
    # stats pass (counters of this rank's slice), not timed
    d = step(pd.STATS)
    stats = dict(d.stats)
    nnz_total = int(d.nnz)
    flags_np = d.flags.cpu().numpy()
    del d
    sampler = ClockSampler(local)
    sampler.start()
    step_ms, cell_ms, launches = [], [], 0
    for _ in range(args.steps):
        flush.fill_(1.0)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        d = step()
        e1.record(stream)
        torch.cuda.synchronize()
        launches += pd.last_launch_count()
        step_ms.append(e0.elapsed_time(e1))
        cell_ms.append(d.stats["ms_cells"])
        del d
    clocks = sampler.stop()
    ms = float(np.mean(step_ms))
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = n / (ms / 1e3) / 1e6

    # ---- e2e through the C ABI: pinned host input (rank 0), host outputs (every rank), copies timed
    e2e_ms = []
    h2d = (hp.numel() * 4 + (0 if hw is None else hw.numel() * 4)) if rank == 0 else 0
    d2h = 0
    for it in range(1 + args.steps):
        flush.fill_(1.0)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        d = step(host=True)
        dt = time.perf_counter() - t0
        d2h = (d.n + 1) * 8 + d.nnz * 8 + d.n * 9
        del d
        if it > 0:
            e2e_ms.append(dt * 1e3)
    e2e_t = float(np.mean(e2e_ms))
    if world > 1:
        t = torch.tensor([e2e_t], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_t = float(t.item())
    e2e_v = n / (e2e_t / 1e3) / 1e6

    # ---- roofline denominators measured on this box, in this job
    fp32_peak = pd.measure_fp32_peak(local) / 1e12   # T lane-ops/s (FFMA chains)
    l2_peak = pd.measure_l2_peak(local) / 1e9        # GB/s (L2-resident reads)

    line = None
    if rank == 0:
        cells_rank = stats["cells"]
        kms = float(np.mean(cell_ms))
        achieved = W_MIN_OPS_PER_CELL * cells_rank / (kms / 1e3) / 1e12
        met = profile_metrics()
        roof = {"bound": "alu", "achieved": achieved, "peak": fp32_peak, "unit": "TFLOP/s",
                "frac": achieved / fp32_peak,
                "traffic": met.get("dram_bytes_per_launch") if met else None,
                "kernel": "cells_kernel (3 capacity tiers, one launch each) + the tier-1 finalize_kernel",
                "kernel_ms": kms, "kernel_share_of_step": kms / ms if world == 1 else None,
                "work_model": "achieved = W_min 2.3e4 FP32 lane-ops/cell (SURVEY.md §8(d)) x cells of this rank / "
                              "cell-kernel time (CUDA events on the launching stream around the tier launches "
                              "and the finalize); peak = FFMA-chain microbenchmark on this GPU in this job "
                              "(pd_measure_fp32_peak); traffic and ncu_* = the tier-1 cells_kernel launch "
                              "(ncu_source)",
                "fp32_peak_measured": fp32_peak, "fp32_peak_nominal": ALU_PEAK_TOPS,
                "l2_peak_measured": l2_peak, "frac_useful": achieved / fp32_peak}
        if met:  # what the counters say (ncu capture of the same code, profiles/)
            dur_s = met["duration_ns"] * 1e-9
            if "fp32_lane_ops" in met:
                roof["frac_fp32_pipe"] = met["fp32_lane_ops"] / dur_s / 1e12 / fp32_peak
            if "lts_bytes" in met:
                roof["frac_l2"] = met["lts_bytes"] / dur_s / 1e9 / l2_peak
            roof["ncu_issue_slot_util"] = met.get("issue_active_pct", 0) / 100.0
            roof["ncu_warps_active"] = met.get("warps_active_pct", 0) / 100.0
            if "threads_per_inst" in met:
                roof["ncu_divergence"] = met["threads_per_inst"] / 32.0
            if "ipc" in met:
                roof["ncu_ipc"] = met["ipc"]
            roof["ncu_dram_gbs"] = met["dram_bytes_per_launch"] / met["duration_ns"]
            roof["ncu_warp_inst_per_cell"] = met["inst_executed"] / met.get("cells", 1e7)
            roof["ncu_source"] = met["_file"]
        cfg = {"workload": f"{wl.name}: {wl.description}", "n": n, "box": list(wl.box),
               "leaf_size": args.leaf or 32, "parallelism": f"seed-sharded x{world}",
               "warm_start": "all" if args.warm_start else ("adaptive" if args.warm_adaptive else "off"),
               "l2": "flushed before every timed step (256 MiB write)", "generation_s": round(gen_s, 1)}
        if world > 1:
            cfg["input"] = "points on rank 0; LBVH NCCL-broadcast, slices exchanged (pd_build_sharded)"
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f64+f32", "data": "synthetic", "config": cfg,
                "roofline": roof,
                "e2e": {"value": e2e_v, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)},
                "clocks": clocks, "gpu_launches": int(launches),
                "stats": {k: stats[k] for k in ("nodes_visited", "leaves_visited", "sites_tested", "clip_tests",
                                                 "clips", "tier_cells", "overflow_cells", "ms_bvh", "ms_cells",
                                                 "ms_csr", "ms_tier", "ms_knn", "faces_dropped",
                                                 "faces_near_degenerate", "degraded_cells")},
                "nnz": nnz_total, "empty_ratio": float(np.mean(flags_np & 1)),
                "step_ms": [round(x, 3) for x in step_ms]}
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(wl)
            line["cpu_reference"] = cpu_reference(wl)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        comm.close()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C4")
    ap.add_argument("--n", type=int, default=None, help="override the config's size (debug only)")
    ap.add_argument("--leaf", type=int, default=0)
    ap.add_argument("--ref-cells", type=int, default=64, help="reference arm: cells per step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--warm-start", action="store_true", help="KNN warm start of every cell (PAPER.md:544-545)")
    ap.add_argument("--warm-adaptive", action="store_true", help="KNN warm start of the dominated sites only")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
