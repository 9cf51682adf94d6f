"""Time pd_build of another checkout (regression hunting): python tools/perf_at.py ROOT [configs...]
Imports ROOT's own binding + pdgen (so its ABI matches its libpd.so); CUDA events, L2 flushed."""
import json
import sys

root = sys.argv[1]
sys.path.insert(0, root)
import numpy as np  # noqa: E402
import torch  # noqa: E402
import pdgen  # noqa: E402
import paper_2605_06408_b200 as pd  # noqa: E402

pd.load_library()
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
for cfg in sys.argv[2:] or ["C4"]:
    wl = pdgen.make(cfg)
    p = torch.from_numpy(wl.points).cuda()
    w = None if wl.weights is None else torch.from_numpy(wl.weights).cuda()
    for _ in range(2):
        d = pd.build_diagram(p, w, wl.box)
        del d
    ms, tiers = [], []
    for _ in range(3):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        d = pd.build_diagram(p, w, wl.box)
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
        tiers.append(d.stats.get("ms_tier"))
        del d
    print(json.dumps({"root": root, "config": cfg, "ms": [round(x, 1) for x in ms], "tiers": tiers[-1]}), flush=True)
    del p, w
    torch.cuda.empty_cache()
