#!/bin/bash
export PYTHONPATH=.
for v in base hm4 hm6; do
  if [ $v = base ]; then unset S1D_LIB_PATH; else export S1D_LIB_PATH=$PWD/build/$v/libswept1d.so; fi
  for wp in "1024 4" "2048 8" "512 4" "256 4" "64 4"; do set -- $wp
    S1D_HEAT_P=$2 timeout 60 python tools/prof_one.py --n 27 --w $1 --steps 2048 --reps 2 | tail -1 | sed "s/^/$v P=$2 /"
  done
done
