#!/bin/bash
# Round profile capture for the bench configuration (run under gpurun, 1 GPU):
#  1. plain bench run (must exit 0)
#  2. ncu launch list of the same command (gpu__time_duration per launch)
#  3. ncu --set full of one Diamond launch (the dominant kernel)
set -e
export PYTHONPATH=.
ARGS=${ARGS:-"--steps 2 --warmup 3 --no-cpu-baseline --no-euler --e2e-steps 1"}
python bench.py $ARGS > gpurun_out/prof_plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py $ARGS > gpurun_out/prof_launches.log 2>&1 || true
python bench.py $ARGS > gpurun_out/prof_plain2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-heat_tile_kernel} -s ${SKIP:-4} -c 1 \
    -o gpurun_out/top_kernel python bench.py $ARGS > gpurun_out/prof_full.log 2>&1 || true
