#!/bin/bash
# A/B the d = 1 gathers: shared-memory ring kernel (k_gather_d1r, R rows) vs register kernel k_gather_d1
python -m pytest tests -m gpu -x -q -k "tet4 or quad4 or d1 or golden" > gpurun_out/t.log 2>&1 || { tail -40 gpurun_out/t.log; exit 1; }
for r in 0 2 3 4 6 0 4; do FEA_D1_MODE=$r timeout 600 python tools/bench_configs.py --configs 3 --runs 5 > gpurun_out/d1r$r.log 2>&1; cat gpurun_out/d1r$r.log >> gpurun_out/d1r_all.log; done
tail -1 gpurun_out/t.log
