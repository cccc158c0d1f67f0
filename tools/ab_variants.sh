#!/bin/bash
# A/B the cfg2 bench over library variants in variants/*.so (one GPU call). Env per variant:
# variants/<name>.env (optional, sourced).
rm -f gpurun_out/ab_*.json
for f in variants/libfea_*.so; do
  n=$(basename $f .so)
  ( [ -f variants/$n.env ] && . variants/$n.env; FEA_LIB_PATH=$f timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 20 > gpurun_out/ab_$n.json 2>&1 )
done
timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 20 > gpurun_out/ab_base.json 2>&1
