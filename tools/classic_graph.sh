#!/bin/bash
# Classic substep loop with / without CUDA-graph replay (dev aid)
export PYTHONPATH=.
for g in 0 1; do
  if [ $g = 1 ]; then export S1D_NO_GRAPHS=1; else unset S1D_NO_GRAPHS; fi
  for n in 16 20 22 27; do
    timeout 120 python tools/prof_one.py --scheme classic --n $n --w 64 --steps ${T:-1024} --reps 2 | tail -1 | sed "s/^/nographs=$g /"
  done
  for m in lengthening flattening; do
    timeout 120 python tools/prof_one.py --eq euler --method $m --scheme classic --n 16 --w 64 --steps 512 --reps 2 | tail -1 | sed "s/^/nographs=$g $m /"
  done
done
