"""One diagram build under compute-sanitizer (tools/sanitize.sh): python tools/sanitize_run.py CFG N [FLAGS]
Env PD_START_TIER / PD_COOP_MIN_V force the cooperative capacity tiers (test knobs of pd_build)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import pdgen  # noqa: E402
import paper_2605_06408_b200 as pd  # noqa: E402

cfg, n = sys.argv[1], int(sys.argv[2])
flags = int(sys.argv[3]) if len(sys.argv) > 3 else 0
wl = pdgen.make(cfg, n=None if n <= 0 else n)
d = pd.build_diagram(wl.points, wl.weights, wl.box, out_host=True, flags=flags)
bx = np.asarray(wl.box, np.float64)
print(cfg, wl.n, "flags", flags, "nnz", d.nnz, "vol/box", float(d.volumes.astype(np.float64).sum() / np.prod(bx[3:] - bx[:3])),
      "tier_cells", d.stats["tier_cells"], flush=True)
