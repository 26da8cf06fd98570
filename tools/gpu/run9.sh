timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu9.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu9.log
python tools/sweep_n.py --n 500000 > gpurun_out/sweep9.txt 2>&1
python tools/sweep_n.py --procs 8 --n 62500 >> gpurun_out/sweep9.txt 2>&1
for v in g16d4 g4d4; do echo $v >> gpurun_out/sweep9.txt; FLOWREC_B200_LIB=paper_2602_15883_b200/_lib_var/$v/libflowrec_b200.so python tools/sweep_n.py --n 500000 >> gpurun_out/sweep9.txt 2>&1; done
cat gpurun_out/sweep9.txt
