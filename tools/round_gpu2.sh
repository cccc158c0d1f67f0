#!/bin/bash
python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1 || { tail -40 gpurun_out/t.log; exit 1; }
timeout 900 python tools/cfg5.py > gpurun_out/cfg5.json 2> gpurun_out/cfg5.err
tail -1 gpurun_out/t.log
