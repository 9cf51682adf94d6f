import sys; import os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, pdgen, paper_2605_06408_b200 as pd
n = int(sys.argv[1]) if len(sys.argv) > 1 else None
wl = pdgen.make("C4", n=n)
p = torch.from_numpy(wl.points).cuda(); w = torch.from_numpy(wl.weights).cuda()
for it in range(2):
    d = pd.build_diagram(p, w, wl.box); torch.cuda.synchronize()
    print(d.stats["ms_tier"], flush=True)
