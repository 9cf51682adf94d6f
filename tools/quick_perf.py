"""Device time of pd_build on the BASELINE configs (iteration tool; the bench line comes from bench.py).

    python tools/quick_perf.py C4 C2 C3 C5 [--flags N] [--reps 3]
Prints one JSON line per config: mean ms (CUDA events, L2 flushed before each build), Mcells/s, per-tier
cell-kernel ms and the work counters.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import pdgen  # noqa: E402
import paper_2605_06408_b200 as pd  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("configs", nargs="*", default=["C4"])
ap.add_argument("--flags", type=int, default=0)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--leaf", type=int, default=0)
a = ap.parse_args()
pd.load_library()
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
for cfg in a.configs:
    wl = pdgen.make(cfg, n=a.n)
    p = torch.from_numpy(wl.points).cuda()
    w = None if wl.weights is None else torch.from_numpy(wl.weights).cuda()
    for _ in range(2):
        d = pd.build_diagram(p, w, wl.box, flags=a.flags, leaf_size=a.leaf)
        del d
    ms, tiers = [], []
    for _ in range(a.reps):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        d = pd.build_diagram(p, w, wl.box, flags=a.flags, leaf_size=a.leaf)
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
        tiers.append(d.stats["ms_tier"])
        del d
    d = pd.build_diagram(p, w, wl.box, flags=a.flags | pd.STATS, leaf_size=a.leaf)
    s = d.stats
    n = wl.n
    print(json.dumps({"config": cfg, "n": n, "ms": round(float(np.mean(ms)), 2), "ms_min": round(min(ms), 2),
                      "mcells_s": round(n / np.mean(ms) / 1e3, 2),
                      "ms_tier": [round(x, 2) for x in np.mean(tiers, axis=0)], "ms_bvh": round(s["ms_bvh"], 2),
                      "ms_csr": round(s["ms_csr"], 2),
                      "per_cell": {k: round(s[k] / n, 2) for k in ("nodes_visited", "leaves_visited", "sites_tested",
                                                                   "clip_tests", "clips")},
                      "tier_cells": s["tier_cells"], "dropped": s["faces_dropped"],
                      "near_degenerate": s["faces_near_degenerate"], "degraded": s["degraded_cells"],
                      "warm_gain": round(s["warm_gain"], 4), "warm": s["warm_start"]}), flush=True)
    del d, p, w
    torch.cuda.empty_cache()
