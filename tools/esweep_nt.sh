#!/bin/bash
# Euler threads-per-CTA probe at large n (dev aid)
export PYTHONPATH=.
for m in lengthening flattening; do for w in ${WS:-256 512 1024}; do for nt in ${NTS:-0 512 1024}; do
  if [ $nt = 0 ]; then unset S1D_EULER_NT; else export S1D_EULER_NT=$nt; fi
  timeout 120 python tools/prof_one.py --eq euler --method $m --n ${N:-22} --w $w --steps ${T:-1024} --reps 2 | tail -1 | sed "s/^/nt=$nt $m /"
done; done; done
