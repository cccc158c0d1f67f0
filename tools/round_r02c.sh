#!/bin/bash
# Final round-2 GPU call: suite, smoke, reference arm, bench line (both timed by wall clock),
# cfg1 graph batches, configs 1-4 (plain and against the oracle), plan / lazy-table traces,
# SpMV, the bench launch list.
set -u
OUT=${OUT:-gpurun_out}
python -m pytest tests -m gpu -q > $OUT/t.log 2>&1; tail -2 $OUT/t.log
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
t0=$SECONDS; python bench.py --impl reference > $OUT/ref.json 2> $OUT/ref.err; echo "reference arm wall $((SECONDS - t0)) s"
t0=$SECONDS; python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench wall $((SECONDS - t0)) s"
python tools/graph_batch.py --configs 1 --branches 1 > $OUT/graph.jsonl 2>&1
python tools/graph_batch.py --configs 1 --branches 4 >> $OUT/graph.jsonl 2>&1
python tools/bench_configs.py --configs 1,2,3,4 --runs 5 > $OUT/configs.jsonl 2> $OUT/configs.err
python tools/bench_configs.py --configs 1,2,3 --runs 5 --oracle > $OUT/configs_oracle.jsonl 2> $OUT/configs_oracle.err
for c in 2 3 5; do python tools/plan_trace.py --config $c --reps 1 --lazy 2> $OUT/lazy_$c.log; done
python tools/bench_spmv.py --configs 1,2,3,4 > $OUT/spmv.jsonl 2> $OUT/spmv.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv \
    --log-file $OUT/launches_bench.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e \
    > $OUT/ncu_bench.log 2>&1
echo round done
