#!/bin/bash
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 80 --csv --log-file gpurun_out/e_launches.csv \
  python bench.py --config E --no-cpu-baseline --steps 1 --warmup 0 --e2e-steps 1 > gpurun_out/e_ncu.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 80 --csv --log-file gpurun_out/d256_launches.csv \
  python bench.py --config D256 --no-cpu-baseline --steps 1 --warmup 0 --e2e-steps 1 > gpurun_out/d256_ncu.log 2>&1
