#!/bin/bash
# A/B tools/bench_configs.py over env settings (one GPU call): $1 = configs
cfgs=${1:-1,2,3,4}
timeout 900 python tools/bench_configs.py --configs $cfgs --runs 3 > gpurun_out/abc_base.log 2>&1
FEA_GATHER_NO_CN=1 timeout 900 python tools/bench_configs.py --configs $cfgs --runs 3 > gpurun_out/abc_nocn.log 2>&1
FEA_GATHER_CN_WIDE=1 timeout 900 python tools/bench_configs.py --configs $cfgs --runs 3 > gpurun_out/abc_cnwide.log 2>&1
FEA_LIB_PATH=variants/libfea_pf3.so timeout 900 python tools/bench_configs.py --configs 2 --runs 3 > gpurun_out/abc_pf3.log 2>&1
