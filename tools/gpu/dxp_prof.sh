#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tcw_dxp_kernel -s 9 -c 1 -o gpurun_out/dxp_full -f \
  python bench.py --config D150 --no-cpu-baseline --steps 1 --warmup 0 --e2e-steps 1 > gpurun_out/dxp_full.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tcw_fwdp_kernel -s 7 -c 1 -o gpurun_out/fwdp_full -f \
  python bench.py --config D150 --no-cpu-baseline --steps 1 --warmup 0 --e2e-steps 1 > gpurun_out/fwdp_full.log 2>&1
echo done
