#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tcw_head_kernel -s 2 -c 1 -o gpurun_out/headE_full -f \
  python bench.py --config E --no-cpu-baseline --steps 1 --warmup 0 --e2e-steps 1 > gpurun_out/headE_full.log 2>&1
echo done
