# round profile pass: default bench line, launch list and one full capture of the epoch kernel
set -x
python bench.py > gpurun_out/fp_bench.json 2> gpurun_out/fp_bench.err; echo bench=$?
python bench.py --local-ranks 8 --steps 10 --no-cpu-baseline > gpurun_out/fp_local8.json 2> gpurun_out/fp_local8.err
ARGS="bench.py --steps 3 --warmup 3 --e2e-steps 2 --no-cpu-baseline"
python $ARGS > gpurun_out/fp_short.json 2> gpurun_out/fp_short.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fp_launches.csv python $ARGS > gpurun_out/fp_ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:jetmlp_epoch -s 3 -c 1 -f -o gpurun_out/fp_epoch_full python $ARGS > gpurun_out/fp_ncu2.log 2>&1
cat gpurun_out/fp_bench.json gpurun_out/fp_local8.json
