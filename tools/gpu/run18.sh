export KIND=unsteady3d ACT=sin REPS=1
python tools/profile_tc.py 200 8 300000 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/e_launches.csv python tools/profile_tc.py 200 8 300000 > gpurun_out/e_ncu.log 2>&1
echo done
