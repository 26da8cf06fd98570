FLOWREC_B200_LIB=paper_2602_15883_b200/_lib_timers/libflowrec_b200.so timeout 300 python tools/phase_times.py > gpurun_out/phases16.txt 2>&1
FLOWREC_B200_LIB=paper_2602_15883_b200/_lib_timers32/libflowrec_b200.so timeout 300 python tools/phase_times.py > gpurun_out/phases32.txt 2>&1
