#!/bin/bash
# P sweep for the heat tile kernel (dev aid)
export PYTHONPATH=.
for w in ${WS:-64 256 1024 2048}; do
  for p in ${PS:-2 4 8 16}; do
    S1D_HEAT_P=$p python tools/prof_one.py --n ${N:-27} --w $w --steps ${T:-1024} --reps 2 2>&1 | tail -1 | sed "s/^/P=$p /"
  done
done
