set -x
python tools/sweep_n.py > gpurun_out/sweep.txt 2>&1
python tools/sweep_n.py --procs 8 --n 62500 >> gpurun_out/sweep.txt 2>&1
ARGS="bench.py --steps 3 --warmup 3 --e2e-steps 2 --no-cpu-baseline"
python $ARGS > gpurun_out/b_plain.json 2> gpurun_out/b_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/C_launches.csv python $ARGS > gpurun_out/ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:jetmlp_epoch -s 3 -c 1 -f -o gpurun_out/epoch_full python $ARGS > gpurun_out/ncu2.log 2>&1
echo done
