timeout 600 python -m pytest tests/test_gpu_distributed_emulated.py -x -q > gpurun_out/pytest_dist.log 2>&1; echo dist=$?
tail -30 gpurun_out/pytest_dist.log
