#!/bin/bash
mkdir -p gpurun_out
out=gpurun_out/ring_ab2.txt
: > $out
export SL_DEBUG_OCC=1
for rep in 1 2; do
  for cv in 0 1; do
    echo "== K2r carveout $cv rep $rep" >> $out
    SL_CARVEOUT=$cv SL_CSR_RING=0 timeout 300 python tools/time_headline.py 100 >> $out 2>&1
    SL_CARVEOUT=$cv SL_CSR_RING=0 timeout 300 python tools/time_d1.py >> $out 2>&1
    echo "== K2q10 carveout $cv rep $rep" >> $out
    SL_CARVEOUT=$cv SL_CSR_RING=1 timeout 300 python tools/time_headline.py 100 >> $out 2>&1
    SL_CARVEOUT=$cv SL_CSR_RING=1 timeout 300 python tools/time_d1.py >> $out 2>&1
  done
done
