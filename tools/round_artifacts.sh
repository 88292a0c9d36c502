#!/bin/bash
# One B200: the round's evidence -- GPU tests, default bench line, ncu launch list of the
# bench command, ncu --set full of one block step's Gram / pivot / F,G update (bench
# schedule; and the Gram alone with the split factorization), the pointwise step kernel,
# a launch trace of one block sweep, Phase-2 timings, and bench lines of the other configs.
#   bash tools/round_artifacts.sh [OUT]      (OUT default gpurun_out/art)
set -u
OUT=${1:-gpurun_out/art}
mkdir -p $OUT
python -m paper_1907_08560_b200.build > /dev/null
python -m pytest tests -m gpu -q -rA > $OUT/pytest_gpu.log 2>&1; tail -2 $OUT/pytest_gpu.log
python bench.py --steps 3 --warmup 3 > $OUT/bench_c3_bo.log 2>&1; tail -c 400 $OUT/bench_c3_bo.log; echo
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_blk -c 3000 --csv \
    --log-file $OUT/launches_bench_bo.csv python bench.py --no-cpu-baseline --warmup 0 --steps 1 > $OUT/ncu_bench.log 2>&1
# bench schedule launch order per block step: gram0 pivot0 upd0 gram1 pivot1 upd1 updZ (k_blk launches 8-10 = step 1, half 0)
ncu --set full --clock-control none --import-source on -k regex:"k_blk_(update|gram|pivot)" -s 7 -c 3 \
    -o $OUT/prof_blk python tools/profile_step.py --variant bo --sweep > $OUT/ncu_full.log 2>&1
GHSVD_SPLIT_FACTOR=1 ncu --set full --clock-control none --import-source on -k regex:"k_blk_(gram|factor)" -s 4 -c 2 \
    -o $OUT/prof_split python tools/profile_step.py --variant bo --sweep > $OUT/ncu_split.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_pair_step -s 2 -c 1 \
    -o $OUT/prof_pw python tools/profile_step.py --kernel 2 --steps 4 > $OUT/ncu_pw.log 2>&1
GHSVD_TRACE=$OUT/trace_c3_sweep1.csv python tools/perf_blocked.py > $OUT/perf_blocked.log 2>&1
python tools/trace_summary.py $OUT/trace_c3_sweep1.csv > $OUT/trace_c3_sweep1.summary.txt
tail -3 $OUT/trace_c3_sweep1.summary.txt
python tools/time_reduce.py --config 3 > $OUT/time_reduce_c3.log 2>&1
python tools/time_reduce.py --config 2 > $OUT/time_reduce_c2.log 2>&1
for c in 0 1 2 5 6; do
  python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline > $OUT/bench_c$c.log 2>&1
done
python bench.py --config 3 --variant pointwise --steps 1 --warmup 3 --no-cpu-baseline > $OUT/bench_c3_pointwise.log 2>&1
ls $OUT
