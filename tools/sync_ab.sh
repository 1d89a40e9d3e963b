#!/bin/bash
# A/B of heat tile-kernel variants selected by an environment knob (round 2:
# S1D_HEAT_SYNC = cta | pair, the since-removed pair-barrier variant; set
# KNOB/MODES for others): heat parity tests per mode, then n = 2^27 swept
# rates per width (dev aid; results under gpurun_out/).
export PYTHONPATH=.
out=${OUT:-gpurun_out/sync_ab.txt}
: > $out
for mode in ${MODES:-cta pair pair512}; do
  if [ -z "$NOTEST" ]; then
    env ${KNOB:-S1D_HEAT_SYNC}=$mode timeout 900 python -m pytest -q -x tests/test_gpu_heat.py tests/test_gpu_fuzz.py \
      "tests/test_gpu_fullsize.py::test_heat_2p27_swept_equals_classic" >> gpurun_out/sync_ab_tests_$mode.log 2>&1
    echo "$mode tests rc=$? $(tail -1 gpurun_out/sync_ab_tests_$mode.log)" >> $out
  fi
  env ${KNOB:-S1D_HEAT_SYNC}=$mode timeout 600 python tools/quick_perf.py ${LOGN:-27} ${WS:-32,64,128,256,512,1024,2048} ${T:-6144} \
    | grep swept | sed "s/^/$mode /" >> $out
done
cat $out
