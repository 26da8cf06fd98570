nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ffma2 tools/probes/ffma2_probe.cu && /tmp/ffma2 > gpurun_out/ffma2.txt 2>&1
python tools/sweep_n.py > gpurun_out/sweep2.txt 2>&1
python tools/sweep_n.py --procs 8 --n 62500 >> gpurun_out/sweep2.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu2.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu2.log
cat gpurun_out/ffma2.txt gpurun_out/sweep2.txt
