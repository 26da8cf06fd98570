timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu6.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu6.log
python tools/sweep_n.py --n 62500,500000 > gpurun_out/sweep6.txt 2>&1
python tools/sweep_n.py --procs 8 --n 62500 >> gpurun_out/sweep6.txt 2>&1
cat gpurun_out/sweep6.txt
