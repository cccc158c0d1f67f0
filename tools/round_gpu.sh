#!/bin/bash
# One GPU call: tests, default bench line, all configs at full size, config 5, launch list and ncu captures
python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1 || { tail -40 gpurun_out/t.log; exit 1; }
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err || exit 1
timeout 900 python tools/bench_configs.py --configs 1,2,3,4 --runs 5 --oracle > gpurun_out/configs.jsonl 2> gpurun_out/configs.err
timeout 900 python tools/cfg5.py > gpurun_out/cfg5.json 2> gpurun_out/cfg5.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1
bash tools/prof_round.sh cfg2_slot:2:sorted:k_gather_slot cfg2_atomic_staged:2:atomic:k_atomic_staged \
    cfg3_d1:3:sorted:k_gather_d1 cfg4_cn:4:sorted:k_gather_cn
tail -1 gpurun_out/t.log
