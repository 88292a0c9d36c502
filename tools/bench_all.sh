#!/bin/bash
# One B200: bench every BASELINE config / variant into gpurun_out/bench_all/ (round table).
set -u
OUT=gpurun_out/bench_all
mkdir -p $OUT
for c in 0 1 2; do
  for v in pointwise bo; do
    python bench.py --config $c --variant $v --no-cpu-baseline > $OUT/bench_c${c}_${v}.log 2>&1
  done
done
python bench.py --config 3 --variant bo --no-cpu-baseline > $OUT/bench_c3_bo.log 2>&1
python bench.py --config 5 --variant bo --no-cpu-baseline > $OUT/bench_c5_bo.log 2>&1
python bench.py --config 5 --variant bo --no-cpu-baseline --want-x > $OUT/bench_c5_bo_x.log 2>&1
python bench.py --config 4 --variant bo --no-cpu-baseline --warmup 1 > $OUT/bench_c4_bo_w1.log 2>&1
for f in $OUT/*.log; do echo "$f $(tail -1 $f | python -c 'import json,sys
try:
  d=json.loads(sys.stdin.read()); print(round(d["value"],4), d["sweeps"], round(d["roofline"]["achieved"],1), round(d["roofline"]["frac"],3))
except Exception as e: print("ERR", e)')"; done
