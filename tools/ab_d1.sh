#!/bin/bash
python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1 || { tail -30 gpurun_out/t.log; exit 1; }
timeout 600 python tools/bench_configs.py --configs 1,2,3,4 --runs 5 --oracle > gpurun_out/configs.jsonl 2>gpurun_out/configs.err
