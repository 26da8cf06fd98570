#!/bin/bash
# round-end style check: full GPU suite, default bench (C + D150 + E nested), C launch list
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/full_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/full_tests.log
python bench.py > gpurun_out/full_bench.json 2> gpurun_out/full_bench.err; echo "bench rc=$?" >> gpurun_out/full_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/full_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/full_tests.log
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv --log-file gpurun_out/full_launches_C.csv \
  python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline --extra-configs "" > gpurun_out/full_ncu.log 2>&1
echo done
