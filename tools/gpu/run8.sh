timeout 300 python -m pytest tests/test_gpu_overlap.py -x -q > gpurun_out/pytest_overlap.log 2>&1; echo overlap=$?
tail -30 gpurun_out/pytest_overlap.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu8.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu8.log
python tools/sweep_n.py --n 500000 > gpurun_out/sweep8.txt 2>&1
cat gpurun_out/sweep8.txt
