#!/bin/bash
# fresh default bench line + launch list; ncu of the d = 1 kernel on the colour route (compare with sorted)
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1
bash tools/prof_round.sh cfg3_d1g_colour:3:colour:k_gather_d1g
cat gpurun_out/bench.json
