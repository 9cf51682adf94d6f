"""Summarize gpurun_out/san_*.log (tools/sanitize.sh) into profiles/<round>_sanitizer.md.
    python tools/sanitize_summary.py r2"""
import glob
import re
import sys

R = sys.argv[1] if len(sys.argv) > 1 else "r2"
lines = [f"# {R}: compute-sanitizer over the cell kernel's capacity tiers (tools/sanitize.sh, SURVEY.md §4 T4)", "",
         "Run on a B200 with `bash tools/sanitize.sh` (each line: one `pd_build` under the tool; `PD_START_TIER` / "
         "`PD_COOP_MIN_V` force every cell into tier 2 or the cooperative top tier with every O(V) pass CTA-wide; "
         "flags 4 = PD_STATS so the tier counts prove which tier ran; flags 32 = PD_WARM_START).  Tier-1 cells are "
         "finalized by finalize_kernel (deferred finalize), which every run with tier-1 cells exercises.", "",
         "| run | tool | env | input | tier_cells (t1, t2, t3) | result |", "|---|---|---|---|---|---|"]
bad = 0
for f in sorted(glob.glob("gpurun_out/san_*.log")):
    if f.endswith("san_all.log"):
        continue
    t = open(f).read()
    m = re.match(r"== (\S+) \((\w+)\) (.*)", t.split("\n")[0])
    if not m:
        continue
    name, tool, cmd = m.groups()
    env = " ".join(x for x in cmd.split() if x.startswith("PD_") and "=" in x) or "-"
    inp = cmd.split("sanitize_run.py")[-1].strip()
    tc = re.search(r"tier_cells (\[[^\]]*\])", t)
    summ = [ln.replace("========= ", "") for ln in t.split("\n") if "SUMMARY" in ln]
    rc = re.search(r"rc=(\d+)", t)
    bad += (rc is None or rc.group(1) != "0")
    lines.append(f"| {name} | {tool} | {env} | {inp} | {tc.group(1) if tc else '?'} | "
                 f"{summ[0] if summ else '?'}; rc={rc.group(1) if rc else '?'} |")
lines += ["", "(tier_cells is counted only with PD_STATS; default-flag runs print [0, 0, 0].)  "
          + ("Every run: 0 errors / 0 hazards." if bad == 0 else f"{bad} run(s) FAILED.")]
open(f"profiles/{R}_sanitizer.md", "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
