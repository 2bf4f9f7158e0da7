#!/bin/bash
# Round evidence on the GPU box: plain bench, ncu launch list, one full ncu
# capture of the first big packed-GEMM pair of the last timed step.
#   bash tools/profile_round.sh <tag>      (outputs in gpurun_out/)
set -u
TAG=${1:-r01}
ARGS="--steps 2 --warmup 3 --no-secondary --no-cpu-baseline --no-general --no-e2e"
mkdir -p gpurun_out
python bench.py $ARGS > gpurun_out/${TAG}_plain.json 2> gpurun_out/${TAG}_plain.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py $ARGS > gpurun_out/${TAG}_ncu_launches.log 2>&1 || exit 2
T=$(grep -c 'dgemm_dmma_kernel' gpurun_out/${TAG}_launches.csv)
SKIP=$((T - 4))
echo "dgemm launches: $T, skipping $SKIP" > gpurun_out/${TAG}_full.log
ncu --set full --clock-control none --import-source on -k regex:dgemm_dmma --launch-skip $SKIP --launch-count 2 \
    -o gpurun_out/${TAG}_full python bench.py $ARGS >> gpurun_out/${TAG}_full.log 2>&1 || exit 3
echo ok
