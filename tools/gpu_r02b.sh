#!/bin/bash
# round-2 call b: forward ablations (K/V load removal, fast engine), event traces, ncu captures
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 bash abl_bin/run.sh
timeout 400 bash tools/gpu_trace.sh
TAG=r02 timeout 2400 bash tools/profile_r02.sh > gpurun_out/profile_r02.log 2>&1
ls -la gpurun_out
