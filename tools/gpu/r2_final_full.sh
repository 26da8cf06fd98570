#!/bin/bash
# full ncu captures of the PDE-set TF32 wide kernels (the MSE-set launches of
# the epoch come first: skip them and the layer-1 launch)
mkdir -p gpurun_out
for c in D150 E; do
  if [ $c = D150 ]; then SK=6; else SK=8; fi
  for k in fwdp dxp dwq head; do
    S=$SK; [ $k = head ] && S=1
    timeout 600 ncu --set full --clock-control none -k regex:tcw_${k}_kernel -s $S -c 1 -f -o /tmp/r2f_${c}_$k \
      python bench.py --config $c --steps 1 --warmup 0 --e2e-steps 1 --no-cpu-baseline > /dev/null 2>&1
    ncu -i /tmp/r2f_${c}_$k.ncu-rep --page raw --csv > gpurun_out/r2f_${c}_$k.raw.csv 2>/dev/null
  done
done
echo done
