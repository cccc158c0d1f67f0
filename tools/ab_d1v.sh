#!/bin/bash
# A/B the d = 1 direct-record gather's batch width U (records one batch ahead) on cfg3; ab_libs/ holds variant builds
FEA_LIB_PATH=ab_libs/libfea_u4.so python -m pytest tests -m gpu -x -q -k "tet4 or quad4 or d1 or golden" > gpurun_out/t.log 2>&1 || { tail -40 gpurun_out/t.log; exit 1; }
python -m pytest tests -m gpu -x -q -k "tet4 or quad4 or d1 or golden" >> gpurun_out/t.log 2>&1 || { tail -40 gpurun_out/t.log; exit 1; }
rm -f gpurun_out/d1g_all.log
for v in default u4 u6 default; do
  if [ $v = default ]; then unset FEA_LIB_PATH; else export FEA_LIB_PATH=ab_libs/libfea_$v.so; fi
  echo "# $v" >> gpurun_out/d1g_all.log
  timeout 600 python tools/bench_configs.py --configs 3 --runs 5 >> gpurun_out/d1g_all.log 2>&1
done
tail -1 gpurun_out/t.log
