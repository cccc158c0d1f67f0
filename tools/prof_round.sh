#!/bin/bash
# ncu --set full captures of the top kernel per case (each case first run once without ncu)
set -u
run() {  # name cfg strategy regex
  python tools/prof_case.py --cfg $2 --strategies $3 --iters 1 > /dev/null || { echo "case $1 failed"; return; }
  ncu --set full --import-source on --clock-control none -k regex:"$4" -c 1 -o gpurun_out/$1 -f \
      python tools/prof_case.py --cfg $2 --strategies $3 --iters 1 > gpurun_out/$1.log 2>&1
  python tools/ncu_summary.py gpurun_out/$1.ncu-rep > gpurun_out/$1.json
  # per-instruction stall table (SASS + source line), small; the report itself only on request
  ncu -i gpurun_out/$1.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/$1.sass.csv.gz
  [ "${KEEP_REP:-0}" = 1 ] || rm -f gpurun_out/$1.ncu-rep
}
for spec in "$@"; do run $(echo $spec | tr ':' ' '); done
