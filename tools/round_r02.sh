#!/bin/bash
# End-of-change GPU call: suite, smoke, default bench line, reference arm, graph batch (cfg1)
set -u
OUT=${OUT:-gpurun_out}
python -m pytest tests -m gpu -q > $OUT/t.log 2>&1; tail -2 $OUT/t.log
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
python bench.py --impl reference > $OUT/ref.json 2> $OUT/ref.err
python bench.py > $OUT/bench.json 2> $OUT/bench.err
tail -c 400 $OUT/bench.err
python tools/graph_batch.py --configs 1 --branches 1 > $OUT/graph.jsonl 2>&1
python tools/graph_batch.py --configs 1 --branches 4 >> $OUT/graph.jsonl 2>&1
python tools/bench_configs.py --configs 1,2,3,4 --runs 5 > $OUT/configs.jsonl 2> $OUT/configs.err
echo done
