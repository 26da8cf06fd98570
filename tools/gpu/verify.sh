set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench_C.json 2> gpurun_out/bench_C.err; echo bench=$?
python bench.py --config D256 --steps 5 --no-cpu-baseline > gpurun_out/bench_D256.json 2> gpurun_out/bench_D256.err; echo benchD=$?
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo benchref=$?
cat gpurun_out/bench_C.json gpurun_out/bench_D256.json gpurun_out/bench_ref.json
