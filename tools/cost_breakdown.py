"""Where the work of a config goes, per cell class (PD_COST work counts; PD_PROF_TIER=0 restricts the
stats to tier 1): EMPTY vs non-empty, degree and cost quantiles.  One JSON line."""
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
d = pd.build_diagram(p, w, wl.box, flags=pd.STATS | pd.COST | int(os.environ.get("FLAGS", "0")))
torch.cuda.synchronize()
s = d.stats
cost = pd.cell_cost(d).cpu().numpy().astype(np.float64)
fl = d.flags.cpu().numpy()
deg = np.diff(d.offsets.cpu().numpy())
emp = (fl & 1) != 0
wts = None if wl.weights is None else wl.weights.astype(np.float64)
out = {"config": cfg, "n": wl.n, "tier_cells": s["tier_cells"],
       "per_cell": {k: round(s[k] / max(s["cells"], 1), 1) for k in ("nodes_visited", "leaves_visited", "sites_tested",
                                                                     "clip_tests", "clips")},
       "empty_frac": float(emp.mean()), "cost_share_empty": float(cost[emp].sum() / cost.sum()),
       "cost_mean_empty": float(cost[emp].mean()) if emp.any() else None,
       "cost_mean_nonempty": float(cost[~emp].mean()),
       "cost_q": [float(np.quantile(cost, q)) for q in (0.5, 0.9, 0.99, 0.999)],
       "deg_mean_nonempty": float(deg[~emp].mean())}
if wts is not None:
    dn = pdgen.median_nn_distance(wl.points)
    z = wts / (dn * dn / 3.0)
    bins = [-np.inf, -10, -3, -1, 1, 3, 10, np.inf]
    idx = np.digitize(z, bins) - 1
    out["by_weight"] = [{"z_range": [bins[k], bins[k + 1]], "frac": float((idx == k).mean()),
                         "cost_share": float(cost[idx == k].sum() / cost.sum()),
                         "empty_frac": float(emp[idx == k].mean()) if (idx == k).any() else None}
                        for k in range(len(bins) - 1)]
print(json.dumps(out, default=lambda x: None if x in (np.inf, -np.inf) else x))
