"""Two C4 builds (N sites, default full C4) for ncu captures: the second build's launches are the profiled ones.
The auto warm-start decision (a sampled tier-1 run with and without the KNN pre-clip) is skipped (it is off on C4
anyway), so the cell-kernel launches of a build are exactly tier 1, tier 2, tier 3 and the tier-1 finalize."""
import sys; import os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, pdgen, paper_2605_06408_b200 as pd
n = int(sys.argv[1]) if len(sys.argv) > 1 else None
wl = pdgen.make("C4", n=n)
p = torch.from_numpy(wl.points).cuda(); w = torch.from_numpy(wl.weights).cuda()
for it in range(2):
    d = pd.build_diagram(p, w, wl.box, flags=pd.NO_AUTO_WARM); torch.cuda.synchronize()
    print(d.stats["ms_tier"], flush=True)
