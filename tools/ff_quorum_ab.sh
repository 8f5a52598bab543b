#!/bin/bash
# A/B of the lane engine's continuous-batching fast-forward gates on config-5 slices (GPU box):
# base (quorum 5/8, FCFS prefill only in the tail), q1 (quorum 1/8), q1fa / q5fa (FCFS prefill always).
# Build first: python tools/ab_build.py base "" q1 "-DSLOSIM_LANE_FF_QUORUM8=1" \
#   q1fa "-DSLOSIM_LANE_FF_QUORUM8=1 -DSLOSIM_LANE_FF_FCFS_ALWAYS" q5fa "-DSLOSIM_LANE_FF_FCFS_ALWAYS"
mkdir -p gpurun_out
for round in 1 2; do
  for v in base q1 q1fa q5fa; do
    SLOSIM_LIB=build/ab/lib_$v.so timeout 300 python tools/variant_time.py 131072 $([ $round = 1 ] && echo parity) 2>&1 | head -2
  done
done
