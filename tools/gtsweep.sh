#!/bin/bash
export PYTHONPATH=.
for meth in lengthening flattening; do for w in 32 64 128 256; do for gt in 1 2 4 8; do
  S1D_EULER_GT=$gt timeout 60 python tools/prof_one.py --eq euler --method $meth --n 22 --w $w --steps 256 --reps 2 | tail -1 | sed "s/^/$meth GT=$gt /"
done; done; done
