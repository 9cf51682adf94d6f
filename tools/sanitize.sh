#!/bin/bash
# GPU box: compute-sanitizer memcheck / racecheck / synccheck / initcheck over the cell kernel's tiers
# (SURVEY.md §4 T4).  Summaries -> gpurun_out/san_*.log
mkdir -p gpurun_out
python -m paper_2605_06408_b200.build > /dev/null
CS="compute-sanitizer --print-limit 20 --error-exitcode 9"
run() {  # name tool env... -- args
  local name=$1 tool=$2; shift 2
  echo "== $name ($tool) $*" > gpurun_out/san_$name.log
  timeout 1500 env "$@" >> gpurun_out/san_$name.log 2>&1
  echo "rc=$?" >> gpurun_out/san_$name.log
}
PY="python tools/sanitize_run.py"
run memcheck_c1 memcheck $CS --tool memcheck $PY C1 0
run memcheck_c5_20k memcheck $CS --tool memcheck $PY C5 20000
run memcheck_c5_tier2 memcheck PD_START_TIER=1 PD_COOP_MIN_V=0 $CS --tool memcheck $PY C5 4000 4
run memcheck_c5_tier3 memcheck PD_START_TIER=2 PD_COOP_MIN_V=0 $CS --tool memcheck $PY C5 3000 4
run memcheck_warm memcheck $CS --tool memcheck $PY C5 8000 32
run racecheck_c1 racecheck $CS --tool racecheck $PY C1 0
run racecheck_c5_tier2 racecheck PD_START_TIER=1 PD_COOP_MIN_V=0 $CS --tool racecheck $PY C5 1500 4
run racecheck_c5_tier3 racecheck PD_START_TIER=2 PD_COOP_MIN_V=0 $CS --tool racecheck $PY C5 600 4
run synccheck_c5_tier3 synccheck PD_START_TIER=2 PD_COOP_MIN_V=0 $CS --tool synccheck $PY C5 1500 4
run synccheck_c1 synccheck $CS --tool synccheck $PY C1 0
run initcheck_c1 initcheck $CS --tool initcheck $PY C1 0
run initcheck_c5_20k initcheck $CS --tool initcheck $PY C5 20000
run memcheck_recfull memcheck PD_REC_CAP=20000 $CS --tool memcheck $PY C4 8000 0
tail -n 4 gpurun_out/san_*.log
