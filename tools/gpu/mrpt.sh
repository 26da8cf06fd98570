#!/bin/bash
mkdir -p gpurun_out
for v in base 3 2; do
  if [ $v = base ]; then L=""; else L="paper_2602_15883_b200/_lib_mr$v/libflowrec_b200.so"; fi
  FLOWREC_B200_LIB=$L python bench.py --local-ranks 8 --steps 10 --no-cpu-baseline > gpurun_out/mr_l8_${v}.json 2>/dev/null
  FLOWREC_B200_LIB=$L python bench.py --steps 20 --no-cpu-baseline --extra-configs "" > gpurun_out/mr_c_${v}.json 2>/dev/null
done
FLOWREC_B200_LIB=paper_2602_15883_b200/_lib_mr3/libflowrec_b200.so python -m pytest tests/test_gpu_kernels.py tests/test_gpu_training.py tests/test_gpu_headline.py tests/test_gpu_tf32x3.py -q -x > gpurun_out/mr_tests.log 2>&1; echo rc=$? >> gpurun_out/mr_tests.log
