# W=64 split-TF32 epoch kernel check: parity tests + config C bench
export FR_PARITY_LOG=gpurun_out/parity.jsonl
timeout 600 python -m pytest tests/test_gpu_tc.py tests/test_gpu_tf32x3.py tests/test_gpu_headline.py -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; tail -3 gpurun_out/gputest.log
timeout 300 python bench.py --steps 10 --warmup 3 --e2e-steps 2 --no-cpu-baseline --extra-configs '' > gpurun_out/bC.json 2> gpurun_out/bC.err
tail -c 600 gpurun_out/bC.json
