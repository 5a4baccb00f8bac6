#!/bin/bash
# ncu evidence for one round (run on the GPU box via gpurun, from the repo root):
#   1. launch list of the bench command (per-launch gpu__time_duration, cold-cache, serialised)
#   2. one `--set full` capture per hot kernel at its 14B shape (scripts/profile_kernels.py)
# Each command first runs once without ncu and must exit 0.
set -e
R=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
WHICH=${WHICH:-"gemm fmha xpb xs conv norm"}   # subset: WHICH="conv xs" LAUNCHES=0 ./scripts/profile_round.sh
if [ "${LAUNCHES:-1}" = 1 ]; then
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/plain_bench.json
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$R.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/ncu_bench.log 2>&1 || true
fi
for w in $WHICH; do
  python scripts/profile_kernels.py $w > /dev/null
done
declare -A K=([gemm]=gemm_tc [fmha]=fmha2 [xpb]=gemm_tc [xs]=gemm_tc [conv]=conv_ [norm]=norm_)
for w in $WHICH; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:${K[$w]} -s 1 -c 1 \
    -o $OUT/full_${R}_$w python scripts/profile_kernels.py $w > $OUT/full_${R}_$w.log 2>&1 || true
done
ls -la $OUT
