#!/bin/bash
mkdir -p gpurun_out
for v in 2 1 3 g; do
  L="paper_2602_15883_b200/_lib_dwu$v/libflowrec_b200.so"
  for i in 1 2; do
    FLOWREC_B200_LIB=$L python bench.py --steps 20 --no-cpu-baseline --extra-configs "" > gpurun_out/dwu_${v}_$i.json 2>/dev/null
  done
done
