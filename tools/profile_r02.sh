#!/bin/bash
# Round-2 profile captures (run under gpurun, 1 GPU; each ncu run only after
# the same command exited 0 without ncu):
#  1. bench (heat headline) launch list (gpu__time_duration per launch)
#  2. ncu --set full of one fast heat Diamond (the dominant kernel)
#  3. ncu --set full of the Euler swept Diamonds and the Euler classic
#     substep kernels (n = 2^22, w = 512)
set -x
export PYTHONPATH=.
ARGS=${ARGS:-"--steps 2 --warmup 3 --no-cpu-baseline --no-euler --e2e-steps 1"}
python bench.py $ARGS > gpurun_out/prof_plain.log 2>&1 || exit 1
[ -n "$SKIP_LAUNCHES" ] || ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py $ARGS > gpurun_out/prof_launches.log 2>&1
# launch order per advance: Up fast, Up gate, Diamond fast, Diamond gate, ...
ncu --set full --clock-control none --import-source on -k regex:heat_tile_kernel -s 2 -c 1 \
    -o gpurun_out/top_kernel -f python bench.py $ARGS > gpurun_out/prof_full.log 2>&1
for m in ${EULER_METHODS-lengthening flattening}; do
  python tools/prof_one.py --eq euler --method $m --n 22 --w 512 --steps 1024 --reps 2 > gpurun_out/prof_e_$m.log 2>&1 || exit 1
  ncu --set full --clock-control none --import-source on -k regex:euler_tile -s 1 -c 1 -o gpurun_out/euler_$m -f \
      python tools/prof_one.py --eq euler --method $m --n 22 --w 512 --steps 1024 --reps 2 > gpurun_out/prof_e_full_$m.log 2>&1
  [ -n "$SKIP_CLASSIC" ] && continue
  python tools/prof_one.py --eq euler --method $m --scheme classic --n 22 --w 512 --steps 128 --reps 2 > gpurun_out/prof_c_$m.log 2>&1 || exit 1
  ncu --set full --clock-control none --import-source on -k "regex:euler_(len|flat)_classic" -s 8 -c 4 \
      -o gpurun_out/classic_$m -f \
      python tools/prof_one.py --eq euler --method $m --scheme classic --n 22 --w 512 --steps 128 --reps 2 > gpurun_out/prof_c_full_$m.log 2>&1
done
ls -la gpurun_out/*.ncu-rep
