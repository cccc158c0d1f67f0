#!/bin/bash
# atomic-route A/B over variants/*.so and the default build
python tools/ab_atomic.py --configs ${CFGS:-2,3} > gpurun_out/ab_atomic_base.jsonl 2>&1
for f in variants/libfea_*.so; do
  FEA_LIB_PATH=$f timeout 300 python tools/ab_atomic.py --configs ${CFGS:-2,3} --staged-only >> gpurun_out/ab_atomic_var.jsonl 2>&1
done
cat gpurun_out/ab_atomic_base.jsonl gpurun_out/ab_atomic_var.jsonl
