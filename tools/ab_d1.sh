#!/bin/bash
# A/B the d = 1 gathers: half-warp slot kernel (default) vs staged-record kernel (FEA_GATHER_NO_SLOT1)
python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1 || { tail -40 gpurun_out/t.log; exit 1; }
timeout 600 python tools/bench_configs.py --configs 1,3 --runs 5 > gpurun_out/d1_slot1.log 2>&1
FEA_GATHER_NO_SLOT1=1 timeout 600 python tools/bench_configs.py --configs 1,3 --runs 5 > gpurun_out/d1_rec.log 2>&1
