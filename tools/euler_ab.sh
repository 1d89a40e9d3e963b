#!/bin/bash
# Euler A/B (dev aid): library variants (VARS: "new" = in-tree, others =
# variants/<v>/libswept1d.so) x methods x schemes at n = 2^N, w, T.
export PYTHONPATH=.
for v in ${VARS:-head new}; do
  if [ $v = new ]; then unset S1D_LIB_PATH; else export S1D_LIB_PATH=$PWD/variants/$v/libswept1d.so; fi
  for meth in lengthening flattening; do
    for w in ${WS:-512}; do
      timeout 300 python tools/prof_one.py --eq euler --method $meth --n ${N:-22} --w $w --steps ${T:-1024} --reps 3 | tail -1 | sed "s/^/$v $meth swept /"
    done
    timeout 300 python tools/prof_one.py --eq euler --method $meth --scheme classic --n ${N:-22} --w 512 --steps ${TC:-128} --reps 3 | tail -1 | sed "s/^/$v $meth classic /"
  done
done
