#!/bin/bash
mkdir -p gpurun_out
cp paper_2409_15097_b200/libbbm.so /tmp/libbbm_real.so
for v in PREP16 PREP32; do
  cp abl_bin/libbbm_$v.so paper_2409_15097_b200/libbbm.so
  timeout 300 python -m pytest tests/test_gpu_prep.py tests/test_gpu_prep_contract.py -x -q > gpurun_out/ps_test_$v.log 2>&1; echo "rc=$?" >> gpurun_out/ps_test_$v.log
done
cp /tmp/libbbm_real.so paper_2409_15097_b200/libbbm.so
timeout 900 bash abl_bin/run.sh
