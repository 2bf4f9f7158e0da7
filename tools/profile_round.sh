#!/bin/bash
# Round evidence on the GPU box (outputs in gpurun_out/):
#   1. plain bench line;
#   2. ncu launch list of the TIMED REGION only (bench.py brackets it with
#      cudaProfilerStart/Stop; --profile-from-start off);
#   3. one `--set full` capture of the first commutator + K2a + K2b launches
#      of the timed region;
#   4. one `--set full` capture of the growth phase's Gram-block kernels
#      (bc_*: one 64-survivor block), which run in setup, not in the window.
#   bash tools/profile_round.sh <tag>
set -u
TAG=${1:-r02}
ARGS="--steps 2 --warmup 3 --no-secondary --no-cpu-baseline --no-general --no-e2e"
mkdir -p gpurun_out
python bench.py $ARGS > gpurun_out/${TAG}_plain.json 2> gpurun_out/${TAG}_plain.err || exit 1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches.csv python bench.py $ARGS > gpurun_out/${TAG}_ncu_launches.log 2>&1 || exit 2
ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:'dgemm|commutator_ah' --launch-count 4 \
    -o gpurun_out/${TAG}_full python bench.py $ARGS > gpurun_out/${TAG}_full.log 2>&1 || exit 3
ncu --set full --clock-control none --import-source on -k regex:'bc_' --launch-skip 30 --launch-count 7 \
    -o gpurun_out/${TAG}_growth python bench.py $ARGS > gpurun_out/${TAG}_growth.log 2>&1 || exit 4
echo ok
