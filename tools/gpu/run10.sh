timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu10.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu10.log
python tools/sweep_n.py --n 500000 > gpurun_out/sweep10.txt 2>&1
python tools/sweep_n.py --procs 8 --n 62500 >> gpurun_out/sweep10.txt 2>&1
cat gpurun_out/sweep10.txt
ARGS="bench.py --steps 3 --warmup 3 --e2e-steps 2 --no-cpu-baseline"
python $ARGS > gpurun_out/b10.json 2> gpurun_out/b10.err && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum --clock-control none -k regex:jetmlp_epoch -s 3 -c 1 --csv python $ARGS > gpurun_out/ncu10.csv 2>&1
grep -E "dram|duration|lts" gpurun_out/ncu10.csv
