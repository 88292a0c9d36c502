#!/bin/bash
# The round's closing evidence on one B200 (after the stored oracle references are in):
# full GPU suite, smoke, the default bench line, the reference arm, config 4's bench line.
#   bash tools/final_evidence.sh [OUT]      (OUT default gpurun_out/final)
set -u
OUT=${1:-gpurun_out/final}
mkdir -p $OUT
python -m paper_1907_08560_b200.build > /dev/null
python -m pytest tests -m gpu -q -rA > $OUT/pytest_gpu.log 2>&1; tail -3 $OUT/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; tail -3 $OUT/smoke.log
python bench.py --steps 3 --warmup 3 > $OUT/bench_c3_bo.log 2>&1; tail -c 600 $OUT/bench_c3_bo.log; echo
python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_reference.log 2>&1; tail -c 400 $OUT/bench_reference.log; echo
python bench.py --config 4 --steps 1 --warmup 3 --no-cpu-baseline > $OUT/bench_c4.log 2>&1; tail -c 300 $OUT/bench_c4.log; echo
python bench.py --config 3 --reduce colpiv --steps 2 --warmup 3 --no-cpu-baseline > $OUT/bench_c3_colpiv.log 2>&1; tail -c 300 $OUT/bench_c3_colpiv.log; echo
