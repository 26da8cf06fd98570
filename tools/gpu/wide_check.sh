# wide-path check: TF32 tests, D150/E benches, D150 launch list with smem metrics
export FR_PARITY_LOG=gpurun_out/parity.jsonl
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_tc.py tests/test_gpu_training.py -m gpu -q -p no:cacheprovider -k 'tf32 or tc or wide' > gpurun_out/gputest.log 2>&1; tail -2 gpurun_out/gputest.log
for c in D150 E; do timeout 300 python bench.py --config $c --steps 5 --warmup 3 --e2e-steps 2 --no-cpu-baseline --extra-configs '' > gpurun_out/bq_$c.json 2>/dev/null; done
CMD="python bench.py --config D150 --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline --extra-configs ''"
eval $CMD > gpurun_out/plain.log 2>&1 && eval ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum --clock-control none -k regex:tcw -c 60 --csv --log-file gpurun_out/launches_d150.csv $CMD > gpurun_out/ncu.log 2>&1
