#!/bin/bash
for v in c6 c8; do FEA_LIB_PATH=variants/libfea_$v.so timeout 600 python tools/bench_configs.py --configs 4 --runs 3 > gpurun_out/slotc_$v.log 2>&1; done
