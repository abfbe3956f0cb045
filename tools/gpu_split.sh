#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 240 python -m pytest tests/test_gpu_attn.py tests/test_gpu_pair.py tests/test_gpu_fullsize.py -x -q > gpurun_out/sp_test.log 2>&1; echo "rc=$?" >> gpurun_out/sp_test.log
timeout 900 bash abl_bin/run.sh
