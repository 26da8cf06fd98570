REPS=1 python tools/profile_tc.py 256 8 500000 && \
REPS=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/d256_launches.csv python tools/profile_tc.py 256 8 500000 > gpurun_out/d256_ncu.log 2>&1
echo done
