"""Load balance of the seed-sharded build, measured on ONE GPU by building each rank's slice in turn:
max/mean of per-slice cell-kernel time = the imbalance a world-N run would see.
Equal-count slices (default) vs cost-balanced slices (PD_BALANCE)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import pdgen  # noqa: E402
import paper_2605_06408_b200 as pd  # noqa: E402

cfgs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["C4", "C5"]
world = int(sys.argv[2]) if len(sys.argv) > 2 else 8
for cfg in cfgs:
    wl = pdgen.make(cfg)
    p = torch.from_numpy(wl.points).cuda()
    w = None if wl.weights is None else torch.from_numpy(wl.weights).cuda()
    for _ in range(2):
        del_ = pd.build_diagram(p, w, wl.box)
        torch.cuda.synchronize()
        del del_
    for name, fl in (("equal_count", 0), ("cost_balanced", pd.BALANCE)):
        per, tot = [], []
        for r in range(world):
            d = pd.build_diagram(p, w, wl.box, shard_rank=r, shard_world=world, flags=fl | pd.STATS)
            torch.cuda.synchronize()
            per.append(d.stats["ms_cells"])
            tot.append(d.stats["ms_total"])
            del d
        per = np.array(per)
        print(json.dumps({"config": cfg, "world": world, "slicing": name, "cells_ms_per_rank": [round(x, 1) for x in per],
                          "max_over_mean": round(float(per.max() / per.mean()), 3),
                          "max_total_ms": round(float(max(tot)), 1)}), flush=True)
