#!/bin/bash
mkdir -p gpurun_out
cp paper_2409_15097_b200/libbbm.so /tmp/libbbm_real.so
cp abl_bin/libbbm_PAIR_INORDER.so paper_2409_15097_b200/libbbm.so
BBM_FWD_KERNEL=pair timeout 240 python -m pytest tests/test_gpu_pair.py -x -q > gpurun_out/io_test.log 2>&1; echo "rc=$?" >> gpurun_out/io_test.log
cp /tmp/libbbm_real.so paper_2409_15097_b200/libbbm.so
BBM_FWD_KERNEL=pair timeout 900 bash abl_bin/run.sh
