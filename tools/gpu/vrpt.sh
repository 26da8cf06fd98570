#!/bin/bash
mkdir -p gpurun_out
for v in 1 2; do
  if [ $v = base ]; then L=""; else L="paper_2602_15883_b200/_lib_vr$v/libflowrec_b200.so"; fi
  FLOWREC_B200_LIB=$L python bench.py --local-ranks 8 --steps 10 --no-cpu-baseline > gpurun_out/vr_${v}.json 2>/dev/null
  FLOWREC_B200_LIB=$L ncu --metrics gpu__time_duration.sum --clock-control none -k regex:jetmlp_kernel -c 16 --csv --log-file gpurun_out/vr_${v}.csv \
     python bench.py --local-ranks 8 --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline > /dev/null 2>&1
done
FLOWREC_B200_LIB=paper_2602_15883_b200/_lib_vr1/libflowrec_b200.so python -m pytest tests/test_gpu_api.py -q -x > gpurun_out/vr_tests.log 2>&1; echo rc=$? >> gpurun_out/vr_tests.log
