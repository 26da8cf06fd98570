timeout 600 python -m pytest tests/test_gpu_ghost_derivatives.py -x -q > gpurun_out/p24.log 2>&1; echo gd=$?
tail -25 gpurun_out/p24.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/p24all.log 2>&1; echo all=$?
tail -3 gpurun_out/p24all.log
python tools/sweep_n.py --n 500000 2>&1 | tail -1
