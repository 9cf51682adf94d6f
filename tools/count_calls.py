"""Measurement helper: per-cell work counters of a PD_STATS build (queue_spills = clip() calls in a
-DPD_COUNT_CALLS library).   PD_LIB=... python tools/count_calls.py C4 [n]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, pdgen, paper_2605_06408_b200 as pd
cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1000000
wl = pdgen.make(cfg, n=n)
p = torch.from_numpy(wl.points).cuda()
w = None if wl.weights is None else torch.from_numpy(wl.weights).cuda()
d = pd.build_diagram(p, w, wl.box, flags=pd.STATS | pd.NO_AUTO_WARM)
s = d.stats
print(cfg, n, {k: round(s[k] / n, 2) for k in ("nodes_visited", "leaves_visited", "sites_tested", "clip_tests", "clips",
                                             "queue_spills")})
