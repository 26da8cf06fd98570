#!/bin/bash
# dW-from-k-quad check: TC tests, TF32 parity tests, D150 / D256 / E bench + launch list + one full capture of dwq
mkdir -p gpurun_out
python -m pytest tests/test_gpu_tc.py tests/test_gpu_kernels.py -q -k "tc or tf32 or tma" > gpurun_out/dwq_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/dwq_tests.log
for c in D150 D256 E; do
  python bench.py --config $c --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/dwq_$c.json 2> gpurun_out/dwq_$c.err
done
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file gpurun_out/dwq_launches_D150.csv \
  python bench.py --config D150 --no-cpu-baseline --steps 1 --warmup 0 --e2e-steps 1 > gpurun_out/dwq_ncu.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tcw_dwq -s 6 -c 1 -o gpurun_out/dwq_full -f \
  python bench.py --config D150 --no-cpu-baseline --steps 1 --warmup 0 --e2e-steps 1 > gpurun_out/dwq_full.log 2>&1
echo done
