#!/bin/bash
mkdir -p gpurun_out
for v in base noconv; do
  if [ $v = base ]; then L=""; else L="paper_2602_15883_b200/_lib_noconv/libflowrec_b200.so"; fi
  FR_TC_DWQ=1 FLOWREC_B200_LIB=$L ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tcw_dw -c 12 --csv --log-file gpurun_out/nc_$v.csv \
      python bench.py --config D150 --no-cpu-baseline --steps 1 --warmup 0 --e2e-steps 1 > /dev/null 2>&1
done
FR_TC_DWQ=0 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tcw_dw -c 12 --csv --log-file gpurun_out/nc_old.csv \
      python bench.py --config D150 --no-cpu-baseline --steps 1 --warmup 0 --e2e-steps 1 > /dev/null 2>&1
