"""Per-tier time and warp-cycle phase split of one build (run under a PD_PROFILE=1 library, PD_LIB=...).

    PD_LIB=paper_2605_06408_b200/libpd_prof.so PD_PROF_TIER=2 python tools/prof_tier.py C5 [n]

Phase counters (warp clock64 cycles summed over the selected tier's warps): init, descend, leaf,
clip, pop, finalize | inside clip: classify, boundary, create, aabb.  Prints one JSON line.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import pdgen  # noqa: E402
import paper_2605_06408_b200 as pd  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
n = int(sys.argv[2]) if len(sys.argv) > 2 else None
wl = pdgen.make(cfg, n=n)
p = torch.from_numpy(wl.points).cuda()
w = None if wl.weights is None else torch.from_numpy(wl.weights).cuda()
FL = int(os.environ.get("FLAGS", "0"))  # extra pd_build flags, e.g. 32 = WARM_START
for _ in range(2):
    d = pd.build_diagram(p, w, wl.box, flags=FL)
    torch.cuda.synchronize()
    del d
d = pd.build_diagram(p, w, wl.box, flags=pd.STATS | pd.COST | FL)
torch.cuda.synchronize()
s = d.stats
names = ["init", "descend", "leaf", "clip", "pop", "finalize", "classify", "boundary", "create", "aabb"]
cyc = {k: v for k, v in zip(names, s.get("warp_cycles", [0] * 10))}
cost = pd.cell_cost(d).cpu().numpy().astype(np.int64)
deg = (d.offsets[1:] - d.offsets[:-1]).cpu().numpy()
top = np.argsort(-cost)[:10]
print(json.dumps({"config": cfg, "n": wl.n, "ms_total": s["ms_total"], "ms_tier": s.get("ms_tier"),
                  "tier_cells": s.get("tier_cells"), "warp_cycles": cyc,
                  "top_cost": [[int(i), int(cost[i]), int(deg[i])] for i in top],
                  "deg_max": int(deg.max()), "deg_p999": float(np.percentile(deg, 99.9))}), flush=True)
print(json.dumps({"stats": {k: s[k] for k in ("cells", "nodes_visited", "leaves_visited", "sites_tested", "clip_tests",
                                              "clips", "queue_spills", "ms_knn")}}), flush=True)
if os.environ.get("PD_TRACE_TOP"):
    # re-run with PD_TRACE_CELL set to each of the costliest cells (kernel printf to stdout)
    for i in top[: int(os.environ["PD_TRACE_TOP"])]:
        os.environ["PD_TRACE_CELL"] = str(int(i))
        d = pd.build_diagram(p, w, wl.box)
        torch.cuda.synchronize()
        del d
