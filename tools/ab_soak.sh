#!/bin/bash
for s in 0.3 0.6 1.5 3; do FEA_BENCH_SOAK_S=$s python bench.py --no-e2e --no-cpu-baseline > gpurun_out/soak_$s.json 2>&1; done
FEA_BENCH_SOAK_S=0.3 python bench.py --no-e2e --no-cpu-baseline --steps 200 > gpurun_out/soak_0.3_200.json 2>&1
