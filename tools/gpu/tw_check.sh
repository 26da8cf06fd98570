#!/bin/bash
# TF32 tensor-width check: wide parity tests + D150 / D256 / E bench lines and launch lists
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -k "tf32 or tc or wide or training or E or d3" > gpurun_out/tw_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/tw_tests.log
for c in D150 D256 E; do
  python bench.py --config $c --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/tw_$c.json 2> gpurun_out/tw_$c.err
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/tw_launches_D150.csv \
  python bench.py --config D150 --no-cpu-baseline --steps 1 --warmup 0 --e2e-steps 1 > gpurun_out/tw_ncu.log 2>&1
echo done
