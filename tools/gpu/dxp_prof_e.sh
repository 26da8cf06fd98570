#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tcw_dxp_kernel -s 10 -c 1 -o gpurun_out/dxpE_full -f \
  python bench.py --config E --no-cpu-baseline --steps 1 --warmup 0 --e2e-steps 1 > gpurun_out/dxpE_full.log 2>&1
echo done
