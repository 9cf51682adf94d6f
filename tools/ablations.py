"""Component ablations on B200 (PAPER.md:874-893 / SURVEY.md §8(f) NEXT-2): slowdown of
isotropic culling, depth-first traversal and the paper-only bounds (no AABB-support
/ exact companions) relative to the default kernel; the diagram is identical in every mode
(tests/test_gpu_parity.py::test_ablations_neutral).  Prints one JSON line per (config, mode)."""
import json
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import pdgen  # noqa: E402
import paper_2605_06408_b200 as pd  # noqa: E402

MODES = {"default": 0, "paper_bound": pd.PAPER_BOUND, "isotropic": pd.ISOTROPIC, "dfs": pd.DFS,
         "no_exact": pd.NO_EXACT, "warm_start": pd.WARM_START}
cfgs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["C2", "C3", "C4"]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
for cfg in cfgs:
    wl = pdgen.make(cfg, n=n)
    p = torch.from_numpy(wl.points).cuda()
    w = None if wl.weights is None else torch.from_numpy(wl.weights).cuda()
    base = None
    for _ in range(6):  # clock ramp-up / memory-pool warm-up before any timed mode
        d = pd.build_diagram(p, w, wl.box)
        torch.cuda.synchronize()
        del d
    for name, fl in MODES.items():
        ts = []
        for it in range(4):
            d = pd.build_diagram(p, w, wl.box, flags=fl | pd.STATS)
            torch.cuda.synchronize()
            if it:
                ts.append(d.stats["ms_total"])
        s = d.stats
        ms = float(np.min(ts))
        base = base or ms
        print(json.dumps({"config": cfg, "n": wl.n, "mode": name, "ms": round(ms, 2), "slowdown": round(ms / base, 3),
                          "nodes_per_cell": round(s["nodes_visited"] / wl.n, 1),
                          "sites_per_cell": round(s["sites_tested"] / wl.n, 1),
                          "tests_per_cell": round(s["clip_tests"] / wl.n, 1),
                          "clips_per_cell": round(s["clips"] / wl.n, 1)}), flush=True)
        del d
