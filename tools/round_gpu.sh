#!/bin/bash
# full GPU suite (release + FEA_DEBUG), smoke, full-size configs 1-4 with the oracle, ncu of the hex27 record kernel
python tools/build_variants.py dbg:-DFEA_DEBUG > /dev/null 2>&1
python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1 || { tail -40 gpurun_out/t.log; exit 1; }
FEA_LIB_PATH=variants/libfea_dbg.so python -m pytest tests -m gpu -x -q > gpurun_out/t_dbg.log 2>&1 || { tail -40 gpurun_out/t_dbg.log; exit 1; }
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1500 python tools/bench_configs.py --configs 1,2,3,4 --runs 3 --oracle > gpurun_out/configs.jsonl 2> gpurun_out/configs.err
bash tools/prof_round.sh r01_ncu_cfg4_gather_cnr:4:sorted:k_gather_cnr
tail -1 gpurun_out/t.log; tail -1 gpurun_out/t_dbg.log; cat gpurun_out/smoke.log
