#!/bin/bash
# the d = 1 ring kernel's ncu capture, then the reference's CPU methods on configs 1-4 (host cores)
bash tools/prof_round.sh r01_ncu_cfg3_gather_d1r:3:sorted:k_gather_d1r
free -g > gpurun_out/free.txt; nproc >> gpurun_out/free.txt; lscpu | grep "Model name" >> gpurun_out/free.txt
timeout 1800 python tools/cpu_ref_configs.py --configs 1,2,3,4 --runs 3 > gpurun_out/cpu_ref.jsonl 2> gpurun_out/cpu_ref.err
cat gpurun_out/free.txt
