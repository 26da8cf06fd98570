#!/bin/bash
mkdir -p gpurun_out
FR_TC_DWQ=1 python tools/dwq_debug.py q1
FR_TC_DWQ=1 python tools/dwq_debug.py q1b
FR_TC_DWQ=0 python tools/dwq_debug.py q0
FR_TC_DWQ=1 FR_TC_FWD=tile FR_TC_DX=tile python tools/dwq_debug.py q1t
FR_TC_DWQ=0 FR_TC_FWD=tile FR_TC_DX=tile python tools/dwq_debug.py q0t
