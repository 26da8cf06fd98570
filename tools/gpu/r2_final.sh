#!/bin/bash
# round-2 final profile pass: bench lines, local-rank proxies, launch lists of C / D150 / E / D256,
# full ncu captures of the wide kernels (D150 and E: fwdp, dxp, dwq, head)
mkdir -p gpurun_out
python bench.py > gpurun_out/r2f_bench.json 2> gpurun_out/r2f_bench.err; echo bench=$?
for n in 2 4 8; do
  python bench.py --local-ranks $n --steps 10 --no-cpu-baseline > gpurun_out/r2f_local$n.json 2> gpurun_out/r2f_local$n.err
done
python bench.py --config D256 --no-cpu-baseline > gpurun_out/r2f_D256.json 2> gpurun_out/r2f_D256.err
ARGS="bench.py --steps 3 --warmup 3 --e2e-steps 2 --no-cpu-baseline --extra-configs ''"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/r2f_launches_C.csv python bench.py --steps 3 --warmup 3 --e2e-steps 2 --no-cpu-baseline --extra-configs "" > /dev/null 2>&1
for c in D150 E D256; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/r2f_launches_$c.csv python bench.py --config $c --steps 1 --warmup 0 --e2e-steps 1 --no-cpu-baseline > /dev/null 2>&1
done
for c in D150 E; do
  for k in fwdp dxp dwq head; do
    timeout 600 ncu --set full --clock-control none -k regex:tcw_${k}_kernel -s 4 -c 1 -f -o /tmp/r2f_${c}_$k \
      python bench.py --config $c --steps 1 --warmup 0 --e2e-steps 1 --no-cpu-baseline > /dev/null 2>&1
    ncu -i /tmp/r2f_${c}_$k.ncu-rep --page raw --csv > gpurun_out/r2f_${c}_$k.raw.csv 2>/dev/null
  done
done
echo done
