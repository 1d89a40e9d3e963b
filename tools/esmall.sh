#!/bin/bash
# Euler small-grid CTA-size probe (dev aid): threads per CTA vs grid size.
export PYTHONPATH=.
for m in lengthening flattening; do for n in 16 18 20 22; do for nt in 256 544 1024; do
  S1D_EULER_NT=$nt timeout 120 python tools/prof_one.py --eq euler --method $m --n $n --w ${W:-512} --steps ${T:-512} --reps 2 | tail -1 | sed "s/^/nt=$nt $m /"
done; done; done
