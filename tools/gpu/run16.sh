timeout 600 python -m pytest tests/test_gpu_distributed_emulated.py tests/test_gpu_overlap.py tests/test_gpu_training.py -x -q > gpurun_out/pytest16.log 2>&1; echo rc=$?
tail -15 gpurun_out/pytest16.log
