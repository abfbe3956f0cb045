#!/bin/bash
# parity of the candidate build, then the same-box A/B (tools/ab.sh)
mkdir -p gpurun_out
cp paper_2409_15097_b200/libbbm.so /tmp/libbbm_real.so
BBM_LIB=$PWD/abl_bin/libbbm_${CAND}.so timeout 300 python -m pytest tests/test_gpu_attn.py tests/test_gpu_pair.py tests/test_gpu_fullsize.py -x -q > gpurun_out/abt_test.log 2>&1; echo "rc=$?" >> gpurun_out/abt_test.log
LIBS="prev $CAND" CONFIGS="${CONFIGS:-c5:binblk c2:binblk c2:dense c4:dense-binblk}" bash tools/ab.sh > /dev/null 2>&1
