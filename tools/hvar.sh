#!/bin/bash
# Variant-library comparison (dev aid): VARS names variants/<v>/libswept1d.so
# ("base" = the in-tree library); WPS lists "w P" pairs.
export PYTHONPATH=.
for v in ${VARS:-base}; do
  if [ $v = base ]; then unset S1D_LIB_PATH; else export S1D_LIB_PATH=$PWD/variants/$v/libswept1d.so; fi
  for wp in ${WPS:-"1024:8" "512:8" "64:8" "32:4"}; do w=${wp%:*}; p=${wp#*:}
    S1D_HEAT_P=$p timeout 120 python tools/prof_one.py --n ${N:-27} --w $w --steps ${T:-6144} --reps 2 | tail -1 | sed "s/^/$v P=$p /"
  done
done
