#!/bin/bash
# A/B the d = 1 gathers: direct-record kernel k_gather_d1g (FEA_D1_DIRECT=U) vs the ring default; pattern probe
python tools/gather_probe_d1.py > gpurun_out/probe_d1.log 2>&1
FEA_D1_DIRECT=4 python -m pytest tests -m gpu -x -q -k "tet4 or quad4 or d1 or golden" > gpurun_out/t.log 2>&1 || { tail -40 gpurun_out/t.log; exit 1; }
rm -f gpurun_out/d1g_all.log
for u in 0 4 8; do
  if [ $u = 0 ]; then unset FEA_D1_DIRECT; else export FEA_D1_DIRECT=$u; fi
  timeout 600 python tools/bench_configs.py --configs 3 --runs 5 >> gpurun_out/d1g_all.log 2>&1
done
tail -1 gpurun_out/t.log
