#!/bin/bash
# GPU box: per-kernel device times (ncu launch list, cold-cache, serialised) of one C4 pd_build at N sites, for each
# library given:   tools/kernel_times.sh N lib1 [lib2 ...]   (lib = base or an ab.py name)
N=$1; shift
for L in "$@"; do
  LIB=paper_2605_06408_b200/libpd.so; [ "$L" != base ] && LIB=paper_2605_06408_b200/libpd_$L.so
  PD_LIB=$LIB ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --kernel-name regex:"cells_kernel|finalize_kernel" python tools/prof_c4n.py $N 2>/dev/null | \
      python3 -c "
import csv,sys,collections
rows=[r for r in csv.reader(sys.stdin) if len(r)>10]
h=rows[0]; acc=collections.defaultdict(list)
for r in rows[1:]:
    d=dict(zip(h,r))
    if d.get('Metric Name')=='gpu__time_duration.sum':
        k=d['Kernel Name']; k=('finalize' if 'finalize' in k else 'tier1' if 'TierCfg<96' in k else 'tier2' if 'TierCfg<384' in k else 'tier3')
        acc[k].append(float(d['Metric Value'])/1e6)
print('$L', {k:[round(x,2) for x in v] for k,v in acc.items()})"
done
