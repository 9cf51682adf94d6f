"""The paper's synthetic workloads on one B200: white noise, density gradient,
K = 5 / 10 Gaussian clusters (sigma 0.1), unweighted and with the paper's weights w ~ N(0, (d_nn^2/3)^2)
(PAPER.md:309-340), at 1M and 10M sites.  Time = pd_build end to end from device-resident input to the
device CSR (BVH + cells + CSR, CUDA events inside the library; median of 5 after 3 warm-ups, the paper's
protocol P:343 with the median reported too).  The paper's H200 "Ours" seconds are quoted beside it as
context (other hardware, FP32-only method): Tab. white noise P:732, gradient P:695, clustered-10 P:621,
clustered-5 P:658, and their weighted versions P:862.

    python tools/paper_sweep.py [sizes=1000000,10000000]  -> one JSON line per (workload, n)
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import pdgen  # noqa: E402
import paper_2605_06408_b200 as pd  # noqa: E402

# H200 seconds at 0.1, 0.5, 1, 2, 5, 10, 15 M (PAPER.md tables, "Ours" rows)
SIZES = [100_000, 500_000, 1_000_000, 2_000_000, 5_000_000, 10_000_000, 15_000_000]
H200 = {
    ("white", False): ([0.017, 0.063, 0.123, 0.227, 0.537, 1.064, 1.582], "P:732"),
    ("gradient", False): ([0.019, 0.071, 0.132, 0.245, 0.561, 1.084, 1.588], "P:695"),
    ("clustered10", False): ([0.456, 0.677, 0.720, 1.027, 1.732, 1.848, 2.530], "P:621"),
    ("clustered5", False): ([0.255, 0.639, 0.598, 1.104, 1.258, 1.914, 2.194], "P:658"),
    ("white", True): ([0.022, 0.067, 0.132, 0.251, 0.612, 1.208, 1.811], "P:862"),
    ("gradient", True): ([0.024, 0.085, 0.142, 0.270, 0.632, 1.233, 1.830], "P:830"),
    ("clustered10", True): ([0.379, 0.685, 0.734, 1.113, 2.071, 2.267, 3.210], "P:768"),
    ("clustered5", True): ([0.284, 0.643, 0.604, 1.162, 1.364, 2.243, 2.879], "P:799"),
}


def points(kind, n, seed):
    if kind == "white":
        return pdgen.white_noise(n, seed)
    if kind == "gradient":
        return pdgen.density_gradient(n, seed)
    return pdgen.clustered(n, seed, k=int(kind[9:]), sigma=0.1)


def main():
    sizes = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [1_000_000, 10_000_000]
    for n in sizes:
        for (kind, weighted), (secs, cite) in H200.items():
            p = points(kind, n, 41)
            w = pdgen.weights_paper(n, pdgen.median_nn_distance(p), 41) if weighted else None
            pt = torch.from_numpy(p).cuda()
            wt = None if w is None else torch.from_numpy(w).cuda()
            ms = []
            for it in range(8):
                d = pd.build_diagram(pt, wt, pdgen.OMEGA_BOX)
                torch.cuda.synchronize()
                if it >= 3:
                    ms.append(d.stats["ms_total"])
                empty = float(torch.mean((d.flags & 1).float()).item())
                del d
            med = float(np.median(ms))
            ref = secs[SIZES.index(n)] if n in SIZES else None
            print(json.dumps({"workload": kind + ("-weighted" if weighted else ""), "n": n, "ms_median": round(med, 2),
                              "ms_mean": round(float(np.mean(ms)), 2), "mcells_s": round(n / med / 1e3, 2),
                              "empty_ratio": round(empty, 4),
                              "paper_h200_s": ref, "paper_cite": cite,
                              "paper_h200_mcells_s": None if ref is None else round(n / ref / 1e6, 2)}), flush=True)
            del pt, wt


if __name__ == "__main__":
    main()
