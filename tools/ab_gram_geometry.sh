#!/bin/bash
# A/B of the block-Gram pipeline geometry (rows per stage x stages) on config 3: rebuilds
# libghsvd.so per variant (GHSVD_NVCC_EXTRA) and times one block sweep with isolated
# kernels (GHSVD_SERIAL=1: t_gram per launch) and whole solves in the bench schedule.
#   bash tools/ab_gram_geometry.sh [OUT]   (restores the default build at the end)
set -u
OUT=${1:-gpurun_out/abg}
mkdir -p $OUT
for v in "32 3" "48 2" "40 2" "16 5" "32 2"; do
  set -- $v
  export GHSVD_NVCC_EXTRA="-DGHSVD_GRAM_RT=$1 -DGHSVD_GRAM_STAGES=$2"
  python -m paper_1907_08560_b200.build --force > /dev/null || { echo "build failed $v"; continue; }
  echo "== RTG $1 stages $2" | tee -a $OUT/ab.log
  GHSVD_SERIAL=1 SWEEPS=1 python tools/perf_blocked.py 2>&1 | tail -1 | tee -a $OUT/ab.log
  python tools/ab_blocked.py --config 3 --reps 2 default 2>&1 | grep variant | tee -a $OUT/ab.log
done
unset GHSVD_NVCC_EXTRA
python -m paper_1907_08560_b200.build --force > /dev/null
