#!/bin/bash
# One GPU call: tests, default bench line, all configs at full size, launch list and ncu captures
python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1 || { tail -40 gpurun_out/t.log; exit 1; }
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err || exit 1
timeout 900 python tools/bench_configs.py --configs 1,2,3,4 --runs 5 --oracle > gpurun_out/configs.jsonl 2> gpurun_out/configs.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1
python tools/prof_case.py --cfg 2 --strategies sorted,colour,atomic --iters 1 > /dev/null && \
ncu --set full --import-source on --clock-control none -k regex:"k_gather_slot|k_scatter" -c 3 -o gpurun_out/cfg2_final \
    python tools/prof_case.py --cfg 2 --strategies sorted,colour,atomic --iters 1 > gpurun_out/ncu_final.log 2>&1
tail -1 gpurun_out/t.log
