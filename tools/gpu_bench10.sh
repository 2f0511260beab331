#!/bin/bash
# ten full bench lines back to back (the driver's N=1 command), for run-to-run spread:
# value, value_cold, e2e and its slowest host step, c2_live bulk host enqueue and pause,
# the 8B live pauses
mkdir -p gpurun_out/bench10
for i in $(seq 1 10); do
  timeout 600 python bench.py > gpurun_out/bench10/b_$i.json 2> gpurun_out/bench10/b_$i.err; echo b_$i=$?
done
