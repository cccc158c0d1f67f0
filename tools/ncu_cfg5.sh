#!/bin/bash
# ncu evidence for the config-5 bench line: --set full captures of the sorted (headline) and
# atomic kernels on config 5, and the launch list (gpu__time_duration) of a short bench run.
# Each command first runs once without ncu.
set -u
OUT=${OUT:-gpurun_out}
python tools/prof_case.py --cfg 5 --strategies sorted,atomic --iters 1 > $OUT/cfg5_case.log 2>&1 || { echo "case failed"; exit 1; }
for spec in sorted:k_gather_slot atomic:k_atomic_patch; do
  s=${spec%%:*}; k=${spec##*:}
  timeout 1200 ncu --set full --import-source on --clock-control none -k regex:$k -c 1 \
      -o $OUT/r02_ncu_cfg5_$s -f python tools/prof_case.py --cfg 5 --strategies $s --iters 1 \
      > $OUT/r02_ncu_cfg5_$s.log 2>&1
  python tools/ncu_summary.py $OUT/r02_ncu_cfg5_$s.ncu-rep > $OUT/r02_ncu_cfg5_$s.json
  ncu -i $OUT/r02_ncu_cfg5_$s.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > $OUT/r02_ncu_cfg5_$s.sass.csv.gz
  rm -f $OUT/r02_ncu_cfg5_$s.ncu-rep
done
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench_plain.json 2>&1 || echo "bench failed"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $OUT/r02_launches_bench.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline \
    > $OUT/ncu_bench.log 2>&1
echo "ncu done"
