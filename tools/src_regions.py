"""Instructions / stall samples per enclosing function (and per labelled block) of pd_cells.cu, from
`ncu -i X --page source --csv --print-source cuda,sass`.   python tools/src_regions.py CSV [cells]

Regions: every function definition of pd_cells.cu starts a region; inside the cell program, `// @region name`
comments start sub-regions (e.g. the descend / pop parts of traverse)."""
import csv
import re
import sys

src = open(sys.argv[3] if len(sys.argv) > 3 else "paper_2605_06408_b200/csrc/pd_cells.cu").read().split("\n")
starts = []
fdef = re.compile(r"^(?:template <[^>]*>\s*)?(?:__device__|__global__)[^;(]*?\b(\w+)\s*\(")
for i, line in enumerate(src, 1):
    m = fdef.match(line)
    if m:
        starts.append((i, m.group(1)))
    m2 = re.search(r"// @region (\S+)", line)
    if m2:
        starts.append((i, m2.group(1)))
starts.sort()


def region(ln):
    name = "(top)"
    for a, nm in starts:
        if a <= ln:
            name = nm
        else:
            break
    return name


cells = float(sys.argv[2]) if len(sys.argv) > 2 else 1e6
hdr = None
fname = None
acc = {}
stall_cols = None
for r in csv.reader(open(sys.argv[1])):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        stall_cols = [k for k in hdr if k.startswith("stall_") and "Not Issued" not in k]
        continue
    if hdr is None or r[0] == "":
        continue
    d = dict(zip(hdr, r))
    try:
        ie = float(d["Instructions Executed"])
        sm = float(d["Warp Stall Sampling (All Samples)"])
    except (ValueError, KeyError):
        continue
    key = region(int(r[0])) if fname == "pd_cells.cu" else fname
    x = acc.setdefault(key, [0.0, 0.0, {}])
    x[0] += ie
    x[1] += sm
    for k in stall_cols:
        try:
            x[2][k] = x[2].get(k, 0.0) + float(d[k])
        except ValueError:
            pass
ti = sum(v[0] for v in acc.values())
ts = sum(v[1] for v in acc.values())
print(f"total {ti / cells:.0f} warp inst/cell")
for k, v in sorted(acc.items(), key=lambda kv: -kv[1][1]):
    top = sorted(v[2].items(), key=lambda kv: -kv[1])[:3]
    tops = " ".join(f"{a[6:]}:{100 * b / max(v[1], 1):.0f}%" for a, b in top)
    print(f"{v[0] / cells:7.0f}/cell {100 * v[0] / ti:5.1f}% inst {100 * v[1] / ts:5.1f}% samples  {k:24s} {tops}")
