export KIND=unsteady3d ACT=sin REPS=1
python tools/profile_tc.py 200 8 100000 && \
ncu --set full --clock-control none --import-source on -k regex:tcw_fwd -s 2 -c 1 -f -o gpurun_out/e_fwd python tools/profile_tc.py 200 8 100000 > gpurun_out/e_fwd.log 2>&1
echo done
