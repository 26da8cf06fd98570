#!/bin/bash
mkdir -p gpurun_out
FLOWREC_B200_LIB=paper_2602_15883_b200/_lib_timers/libflowrec_b200.so timeout 300 python tools/phase_times.py > gpurun_out/phases_tc.txt 2>&1
