"""GPU-vs-oracle comparator (SURVEY.md §8(c) "Comparator", BASELINE.json north_star tolerances).

Per checked cell i:
  * neighbour sets must be equal, except pairs present on one side only whose area on the side that
    has them is below tau_ij = 1e-9 * max(S_i, S_j) (symmetric excusal);
    excused pairs are counted and reported;
  * |vol_gpu - vol_oracle| <= 1e-4 * vol_oracle (cells not excused);
  * |a_gpu - a_oracle| <= 1e-3 * a_oracle for every pair not excused;
  * an EMPTY-flag mismatch is excused only if every face of the non-empty side is below tau;
  * the BOUNDARY (a wall face of area > 1e-13 S, reading R3) and DUPLICATE (reading R5) flags must
    be equal.
The oracle's near-degenerate counts (bisector faces <= 1e-13 S it drops, neighbour faces < 1e-9 S)
are summed into the report beside the GPU's (pd_stats faces_dropped / faces_near_degenerate).
S_i comes from the oracle; S_j from the oracle when j was checked, else from the GPU output.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

TAU_REL = 1e-9
VOL_REL = 1e-4
AREA_REL = 1e-3
EMPTY, BOUNDARY, DUPLICATE = 1, 2, 8


@dataclass
class Report:
    cells: int = 0
    passed: int = 0
    excused_pairs: int = 0
    max_rel_area: float = 0.0
    max_rel_vol: float = 0.0
    flag_checked: int = 0
    oracle_dropped: int = 0
    oracle_small: int = 0
    failures: list = field(default_factory=list)

    @property
    def ok(self) -> bool:
        return self.passed == self.cells

    def summary(self) -> str:
        return (f"cells={self.cells} passed={self.passed} excused_pairs={self.excused_pairs} "
                f"max_rel_area={self.max_rel_area:.3g} max_rel_vol={self.max_rel_vol:.3g} "
                f"flags_checked={self.flag_checked} oracle_dropped={self.oracle_dropped} "
                f"oracle_small={self.oracle_small} "
                f"first_failures={self.failures[:5]}")


def compare(gpu, orc, max_failures: int = 50) -> Report:
    """gpu: numpy Diagram (full original-order CSR); orc: oracle.OracleCells for orc.ids."""
    rep = Report()
    g_off, g_nbr, g_area = np.asarray(gpu.offsets), np.asarray(gpu.neighbors), np.asarray(gpu.areas)
    g_vol, g_surf, g_flags = np.asarray(gpu.volumes), np.asarray(gpu.surface), np.asarray(gpu.flags)
    o_surf = {int(i): float(s) for i, s in zip(orc.ids, orc.surf)}
    for t, i in enumerate(orc.ids):
        i = int(i)
        rep.cells += 1
        on, oa = orc.row(t)
        gn = g_nbr[g_off[i]:g_off[i + 1]]
        ga = g_area[g_off[i]:g_off[i + 1]].astype(np.float64)
        S_i = float(orc.surf[t])
        od = dict(zip(on.tolist(), oa.tolist()))
        gd = dict(zip(gn.tolist(), ga.tolist()))
        ok = True
        why = []
        if len(gn) and np.any(np.diff(gn) <= 0):
            ok = False
            why.append("row not strictly ascending")
        if i in gd:
            ok = False
            why.append("self in row")
        for j in set(od) ^ set(gd):
            a = od.get(j, gd.get(j))
            S_j = o_surf.get(j, float(g_surf[j]) if j < len(g_surf) else 0.0)
            if a < TAU_REL * max(S_i, S_j):
                rep.excused_pairs += 1
            else:
                ok = False
                why.append(f"nbr {j} only in {'oracle' if j in od else 'gpu'} (area {a:.3g}, S {S_i:.3g})")
        for j in set(od) & set(gd):
            a, b = od[j], gd[j]
            S_j = o_surf.get(j, float(g_surf[j]))
            if a < TAU_REL * max(S_i, S_j):
                continue
            rel = abs(a - b) / a
            rep.max_rel_area = max(rep.max_rel_area, rel)
            if rel > AREA_REL:
                ok = False
                why.append(f"area {j}: {b} vs {a}")
        same_empty = bool(orc.flags[t] & EMPTY) == bool(g_flags[i] & EMPTY)
        for bit, nm in ((BOUNDARY, "BOUNDARY"), (DUPLICATE, "DUPLICATE")):
            if bit == BOUNDARY and not same_empty:  # an excused EMPTY mismatch (below) decides these cells
                continue
            if bool(orc.flags[t] & bit) != bool(g_flags[i] & bit):
                ok = False
                why.append(f"{nm} flag oracle={bool(orc.flags[t] & bit)} gpu={bool(g_flags[i] & bit)}")
        rep.flag_checked += 1
        if getattr(orc, "dropped", None) is not None:
            rep.oracle_dropped += int(orc.dropped[t])
            rep.oracle_small += int(orc.small[t])
        o_empty = bool(orc.flags[t] & EMPTY)
        g_empty = bool(g_flags[i] & EMPTY)
        if o_empty != g_empty:
            faces = oa if not o_empty else ga
            if not np.all(faces < TAU_REL * max(S_i, 1e-300)):
                ok = False
                why.append(f"EMPTY mismatch oracle={o_empty} gpu={g_empty}")
        else:
            vo, vg = float(orc.vol[t]), float(g_vol[i])
            if vo > 0:
                rel = abs(vg - vo) / vo
                rep.max_rel_vol = max(rep.max_rel_vol, rel)
                if rel > VOL_REL:
                    ok = False
                    why.append(f"vol {vg} vs {vo}")
            elif vg != 0:
                ok = False
                why.append(f"vol {vg} for an empty cell")
        if ok:
            rep.passed += 1
        elif len(rep.failures) < max_failures:
            rep.failures.append((i, why[:4]))
    return rep


def sample_cells(gpu, n: int, seed: int, n_random: int = 256, n_stratum: int = 64, cost=None) -> np.ndarray:
    """Parity sample: random cells + the cost tail (the largest per-cell GPU work,
    pd_cell_cost, when given; else the largest rows) + BOUNDARY + EMPTY cells + every OVERFLOW cell."""
    rng = np.random.default_rng(seed)
    flags = np.asarray(gpu.flags)
    tail = np.asarray(cost) if cost is not None else np.diff(np.asarray(gpu.offsets))
    picks = [rng.choice(n, size=min(n_random, n), replace=False)]
    picks.append(np.argsort(-tail, kind="stable")[:n_stratum])
    for bit in (2, 1):
        idx = np.flatnonzero(flags & bit)
        if len(idx):
            picks.append(rng.choice(idx, size=min(n_stratum, len(idx)), replace=False))
    picks.append(np.flatnonzero(flags & 4))
    return np.unique(np.concatenate(picks)).astype(np.int64)
