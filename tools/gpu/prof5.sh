ARGS="bench.py --steps 3 --warmup 3 --e2e-steps 2 --no-cpu-baseline"
python $ARGS > gpurun_out/b11.json 2> gpurun_out/b11.err && \
ncu --set full --clock-control none --import-source on -k regex:jetmlp_epoch -s 3 -c 1 -f -o gpurun_out/epoch_full11 python $ARGS > gpurun_out/ncu11.log 2>&1
cat gpurun_out/b11.json
