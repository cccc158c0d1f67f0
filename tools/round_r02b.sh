#!/bin/bash
# Round-2 refresh after the lane-owned d = 1 gather and the ticketed / tiled atomic patches:
# suite, smoke, reference arm, bench line, cfg1 graph batches, configs 1-4 with the oracle,
# ncu --set full of the cfg3 gather, the bench launch list.
set -u
OUT=${OUT:-gpurun_out}
bash tools/round_r02.sh
python tools/bench_configs.py --configs 1,2,3 --runs 5 --oracle > $OUT/configs_oracle.jsonl 2> $OUT/configs_oracle.err
bash tools/prof_round.sh cfg3_d1s_rec4:3:sorted:k_gather_d1s cfg3_d1s_colour:3:colour:k_gather_d1s
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $OUT/r02b_launches_bench.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e \
    > $OUT/ncu_bench.log 2>&1
echo refresh done
