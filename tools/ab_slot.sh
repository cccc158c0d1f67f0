#!/bin/bash
# A/B the lane = slot gather (default for d in 2..4, npe in {4,8}) against the column-node kernel
python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1 || { tail -40 gpurun_out/t.log; exit 1; }
timeout 600 python tools/bench_configs.py --configs 2 --runs 5 > gpurun_out/slot_new.log 2>&1
for v in $(ls variants | sed 's/libfea_//; s/.so//'); do
  FEA_LIB_PATH=variants/libfea_$v.so timeout 600 python tools/bench_configs.py --configs 2 --runs 5 > gpurun_out/slot_$v.log 2>&1; done
python bench.py --no-e2e --no-cpu-baseline > gpurun_out/bench_slot.json 2>&1
