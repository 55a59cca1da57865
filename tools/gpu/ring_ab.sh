#!/bin/bash
# A/B: CSR register hand-off (K2r) vs the two-stage ring (K2q) on the
# headline stencil and D1, plus CSR/COO parity under the ring.
mkdir -p gpurun_out
out=gpurun_out/ring_ab.txt
: > $out
for rep in 1 2; do
  echo "== K2r rep $rep" >> $out
  SL_CSR_RING=0 timeout 300 python tools/time_headline.py 100 >> $out 2>&1
  SL_CSR_RING=0 timeout 300 python tools/time_d1.py >> $out 2>&1
  for b in 10 9 8; do
    echo "== K2q blocks $b rep $rep" >> $out
    SL_CSR_RING=1 SL_CSR_RING_BLOCKS=$b timeout 300 python tools/time_headline.py 100 >> $out 2>&1
    SL_CSR_RING=1 SL_CSR_RING_BLOCKS=$b timeout 300 python tools/time_d1.py >> $out 2>&1
  done
done
SL_CSR_RING=1 timeout 600 python -m pytest tests -m gpu -x -q -k "csr or coo or spmv or smoke" > gpurun_out/ring_parity.log 2>&1
echo "parity rc=$?" >> $out
tail -2 gpurun_out/ring_parity.log >> $out
