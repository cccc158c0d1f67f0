#!/bin/bash
# memory-safety pass: every GPU test and every route of tools/sanitize_case.py on the -DFEA_DEBUG bounds-trap build
python tools/build_variants.py dbg:-DFEA_DEBUG > /dev/null 2>&1
FEA_LIB_PATH=variants/libfea_dbg.so python -m pytest tests -m gpu -x -q > gpurun_out/t_dbg.log 2>&1 || { tail -40 gpurun_out/t_dbg.log; exit 1; }
FEA_LIB_PATH=variants/libfea_dbg.so timeout 900 python tools/sanitize_case.py > gpurun_out/sanitize.log 2>&1; echo "sanitize rc=$?" >> gpurun_out/sanitize.log
tail -1 gpurun_out/t_dbg.log; tail -3 gpurun_out/sanitize.log
