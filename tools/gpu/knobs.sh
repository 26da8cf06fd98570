#!/bin/bash
mkdir -p gpurun_out
for v in base v6 ve; do
  if [ $v = base ]; then L=""; else L="paper_2602_15883_b200/_lib_$v/libflowrec_b200.so"; fi
  for i in 1 2; do
    FLOWREC_B200_LIB=$L python bench.py --steps 20 --no-cpu-baseline --extra-configs "" > gpurun_out/kn_${v}_$i.json 2>/dev/null
  done
done
