#!/bin/bash
# tools/ab_time.py over the default build and variants/*.so (+ optional variants/<name>.env): CFGS, STRAT env
python tools/ab_time.py --configs ${CFGS:-4} --strategy ${STRAT:-sorted}
for f in variants/libfea_*.so; do
  n=$(basename $f .so)
  ( [ -f variants/$n.env ] && . variants/$n.env; FEA_LIB_PATH=$f timeout 300 python tools/ab_time.py --configs ${CFGS:-4} --strategy ${STRAT:-sorted} )
done
python tools/ab_time.py --configs ${CFGS:-4} --strategy ${STRAT:-sorted}
