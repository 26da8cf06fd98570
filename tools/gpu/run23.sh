python tools/sweep_n.py --n 500000 2>&1 | tail -1
ARGS="tools/sweep_n.py --n 500000"
ncu --metrics launch__occupancy_limit_shared_mem,launch__occupancy_limit_registers,sm__warps_active.avg.pct_of_peak_sustained_active,launch__shared_mem_per_block_dynamic,gpu__time_duration.sum --clock-control none -k regex:jetmlp_epoch -c 1 --csv python $ARGS 2>&1 | grep -E "occupancy|warps_active|shared_mem|duration" | sed 's/.*Command line profiler metrics//'
