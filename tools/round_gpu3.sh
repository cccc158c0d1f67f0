#!/bin/bash
# full GPU suite (release + FEA_DEBUG bounds-trap build), then full-size configs 1-4 with the oracle
python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1 || { tail -40 gpurun_out/t.log; exit 1; }
FEA_LIB_PATH=variants/libfea_dbg.so python -m pytest tests -m gpu -x -q > gpurun_out/t_dbg.log 2>&1 || { tail -40 gpurun_out/t_dbg.log; exit 1; }
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1500 python tools/bench_configs.py --configs 1,2,3,4 --runs 3 --oracle > gpurun_out/configs.jsonl 2> gpurun_out/configs.err
tail -1 gpurun_out/t.log; tail -1 gpurun_out/t_dbg.log; cat gpurun_out/smoke.log
