#!/bin/bash
# ncu launch list of the bench command (block 6 of the timed rollout), final build.
export PYTHONPATH=$PWD
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/block6/" --csv --log-file gpurun_out/rf_launch.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/rf_launch.log 2>&1; echo ncu rc=$?
