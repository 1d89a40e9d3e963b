#!/bin/bash
# Euler perf sweep (dev aid): classic vs swept across widths
export PYTHONPATH=.
for meth in ${METHODS:-lengthening flattening}; do
  python tools/prof_one.py --eq euler --method $meth --scheme classic --n ${N:-22} --w 64 --steps ${TC:-64} --reps 2 2>&1 | tail -1 | sed "s/^/$meth /"
  for w in ${WS:-64 128 256 512 1024}; do
    python tools/prof_one.py --eq euler --method $meth --n ${N:-22} --w $w --steps ${T:-512} --reps 2 2>&1 | tail -1 | sed "s/^/$meth /"
  done
done
