"""CPU reference of the same definition on full configs, on the host cores:
    python tools/cpu_reference.py C2 [C1 ...] >> profiles/r2_cpu_reference.jsonl
Each line: Mcells/s over the FULL diagram (k-d tree build included), threads, and its agreement with the
brute-force oracle on a 2000-cell sample (comparator of tests/compare.py)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import oracle  # noqa: E402
import pdgen  # noqa: E402
from compare import compare  # noqa: E402


class _D:
    pass


for cfg in sys.argv[1:] or ["C2"]:
    wl = pdgen.make(cfg)
    th = os.cpu_count() or 1
    t = time.time()
    k = oracle.cells(wl.points, wl.weights, wl.box, threads=th, kdtree=True)
    dt = time.time() - t
    ids = np.random.default_rng(5).choice(wl.n, size=min(wl.n, 2000), replace=False)
    o = oracle.cells(wl.points, wl.weights, wl.box, ids=ids, threads=th)
    d = _D()
    d.offsets, d.neighbors, d.areas, d.volumes, d.surface, d.flags = k.offsets, k.nbr, k.area, k.vol, k.surf, k.flags
    rep = compare(d, o)
    print(json.dumps({"config": cfg, "n": wl.n, "seconds": round(dt, 2), "mcells_s": wl.n / dt / 1e6, "threads": th,
                      "cpu": os.popen("lscpu | grep 'Model name' | head -1").read().split(":")[-1].strip(),
                      "oracle_sample_check": rep.summary()[:120]}), flush=True)
