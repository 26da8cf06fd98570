#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/ref_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/ref_tests.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 --cpu-scaling-epochs 1 > gpurun_out/ref_arm.json 2> gpurun_out/ref_arm.err; echo "ref rc=$?" >> gpurun_out/ref_tests.log
python bench.py --extra-configs "" > gpurun_out/ref_ours.json 2> gpurun_out/ref_ours.err; echo "ours rc=$?" >> gpurun_out/ref_tests.log
