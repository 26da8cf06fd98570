timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest_full.log 2>&1; echo full=$?
tail -30 gpurun_out/pytest_full.log
