"""Runtime vs weight magnitude / empty ratio (the paper's table at, run on
its real "bicycle" scene, 0.595 s -> 2.243 s as the empty ratio goes 0 -> 0.468).  Here: the scene-like C4 positions
(10M) with the paper's weight law scaled by s, w ~ N(0, (s d_nn^2/3)^2) (the
paper's "weight ratio" unit is not recoverable from its text, SURVEY.md §8(c) Q13 / DESIGN.md R16), so s is swept
until the empty ratio passes the paper's 0.47.  Each s is timed with the default options and with PD_AUTO_WARM
(the sampled warm-start decision); time = pd_build end to end (ms_total, CUDA events in the library), median of 5 after 3 warm-ups.

    python tools/weight_sweep.py [n=10000000]  -> one JSON line per (s, mode)
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import pdgen  # noqa: E402
import paper_2605_06408_b200 as pd  # noqa: E402

PAPER = [(0.0, 0.000, 0.595), (1e-6, 0.000, 0.596), (1e-5, 4.524e-6, 0.596), (1e-4, 7.726e-4, 0.598),
         (1e-3, 0.051, 0.808), (1e-2, 0.250, 1.469), (1e-1, 0.468, 2.243)]  # (ratio, empty, s) PAPER.md:571-577


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
    pts = pdgen.scene_like(n, 4)
    d_nn = pdgen.median_nn_distance(pts, 4)
    pt = torch.from_numpy(pts).cuda()
    for s in [0.0, 1.0, 3.0, 10.0, 30.0, 100.0, 300.0, 1000.0]:
        w = pdgen.weights_paper(n, d_nn, 4, ratio=s) if s > 0 else None
        wt = None if w is None else torch.from_numpy(w).cuda()
        for mode, flags in (("default", 0), ("auto_warm", pd.AUTO_WARM)):
            ms = []
            for it in range(8):
                d = pd.build_diagram(pt, wt, pdgen.OMEGA_BOX, flags=flags)
                torch.cuda.synchronize()
                if it >= 3:
                    ms.append(d.stats["ms_total"])
                st = d.stats
                flags_t = d.flags
                del d
            empty = float(torch.mean((flags_t & 1).float()).item())
            isolated = None
            print(json.dumps({"workload": "C4 scene-like positions", "n": n, "s": s, "mode": mode,
                              "ms_median": round(float(np.median(ms)), 2), "mcells_s": round(n / np.median(ms) / 1e3, 2),
                              "empty_ratio": round(empty, 4), "isolated_ratio": isolated,
                              "warm_gain": round(st["warm_gain"], 4), "warm_start": st["warm_start"],
                              "ms_tier": [round(x, 2) for x in st["ms_tier"]], "paper_table": PAPER}), flush=True)
            if s == 0:
                break
        del wt
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
