#!/bin/bash
# Euler variant-library comparison (dev aid): VARS names variants/<v>/libswept1d.so
# ("base" = the in-tree library).
export PYTHONPATH=.
for v in ${VARS:-base}; do
  if [ $v = base ]; then unset S1D_LIB_PATH; else export S1D_LIB_PATH=$PWD/variants/$v/libswept1d.so; fi
  for m in lengthening flattening; do for nw in ${NWS:-"22:512" "22:128" "16:512"}; do n=${nw%:*}; w=${nw#*:}
    timeout 120 python tools/prof_one.py --eq euler --method $m --n $n --w $w --steps ${T:-1024} --reps 2 | tail -1 | sed "s/^/$v $m /"
  done; done
done
