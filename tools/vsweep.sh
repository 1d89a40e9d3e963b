#!/bin/bash
export PYTHONPATH=.
for wp in ${WPS:-"1024 4" "1024 8" "2048 8" "256 4" "64 4" "64 2"}; do set -- $wp
  for v in ${VS:-1 2 4}; do
    S1D_HEAT_V=$v S1D_HEAT_P=$2 timeout 60 python tools/prof_one.py --n 27 --w $1 --steps 2048 --reps 2 | tail -1 | sed "s/^/V=$v P=$2 /"
  done
done
