#!/bin/bash
# end-of-session check: GPU suite, smoke, default bench line, reference arm, launch list, config 5
python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1 || { tail -40 gpurun_out/t.log; exit 1; }
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1
timeout 900 python tools/cfg5.py > gpurun_out/cfg5.json 2> gpurun_out/cfg5.err
tail -1 gpurun_out/t.log; cat gpurun_out/smoke.log; cat gpurun_out/bench.json; cat gpurun_out/cfg5.json
