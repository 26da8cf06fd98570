#!/bin/bash
mkdir -p gpurun_out
for v in 4 2 3; do
  if [ $v = 4 ]; then L=""; else L="paper_2602_15883_b200/_lib_hns$v/libflowrec_b200.so"; fi
  for c in E D150; do
    FLOWREC_B200_LIB=$L ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tcw_head -c 4 --csv --log-file gpurun_out/hns_${v}_$c.csv \
      python bench.py --config $c --no-cpu-baseline --steps 1 --warmup 0 --e2e-steps 1 > /dev/null 2>&1
  done
done
