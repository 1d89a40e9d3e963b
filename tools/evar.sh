#!/bin/bash
export PYTHONPATH=.
for v in base mb3 mb4; do
  if [ $v = base ]; then unset S1D_LIB_PATH; else export S1D_LIB_PATH=$PWD/build/var_$v/libswept1d.so; fi
  for nt in 256 128; do
    S1D_EULER_NT=$nt python tools/prof_one.py --eq euler --n 22 --w 512 --steps 512 --reps 2 | tail -1 | sed "s/^/$v nt=$nt /"
    S1D_EULER_NT=$nt python tools/prof_one.py --eq euler --n 22 --w 128 --steps 256 --reps 2 | tail -1 | sed "s/^/$v nt=$nt /"
  done
  python tools/prof_one.py --eq euler --scheme classic --n 22 --w 64 --steps 32 --reps 2 | tail -1 | sed "s/^/$v /"
  python tools/prof_one.py --eq euler --method flattening --scheme classic --n 22 --w 64 --steps 32 --reps 2 | tail -1 | sed "s/^/$v flat /"
done
