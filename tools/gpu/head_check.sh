#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests/test_gpu_tc.py tests/test_gpu_kernels.py tests/test_gpu_training.py -q -k "tc or tf32 or tma or wide or d3" > gpurun_out/head_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/head_tests.log
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:tcw_head -c 6 --csv --log-file gpurun_out/head_launches.csv \
  python bench.py --config E --no-cpu-baseline --steps 1 --warmup 0 --e2e-steps 1 > gpurun_out/head_ncu.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:tcw_head -c 6 --csv --log-file gpurun_out/head_launches_d150.csv \
  python bench.py --config D150 --no-cpu-baseline --steps 1 --warmup 0 --e2e-steps 1 > gpurun_out/head_ncu2.log 2>&1
