#!/bin/bash
# GPU suite (release + FEA_DEBUG) after the d = 1 direct-record kernel, cfg1/3 full size with the oracle, ncu of the kernel
python tools/build_variants.py dbg:-DFEA_DEBUG > /dev/null 2>&1 || true
python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1 || { tail -40 gpurun_out/t.log; exit 1; }
FEA_LIB_PATH=variants/libfea_dbg.so python -m pytest tests -m gpu -x -q -k "tet4 or quad4 or d1 or golden or partition" > gpurun_out/t_dbg.log 2>&1 || { tail -40 gpurun_out/t_dbg.log; exit 1; }
timeout 900 python tools/bench_configs.py --configs 1,3 --runs 5 --oracle > gpurun_out/configs13.jsonl 2> gpurun_out/configs13.err
bash tools/prof_round.sh r01_ncu_cfg3_gather_d1g:3:sorted:k_gather_d1g
tail -1 gpurun_out/t.log; tail -1 gpurun_out/t_dbg.log
