mkdir -p gpurun_out
cp paper_2409_15097_b200/libbbm.so /tmp/libbbm_real.so
cp abl_bin/libbbm_PARTS4.so paper_2409_15097_b200/libbbm.so
timeout 240 python -m pytest tests/test_gpu_attn.py -x -q > gpurun_out/p4_test.log 2>&1; echo "rc=$?" >> gpurun_out/p4_test.log
cp /tmp/libbbm_real.so paper_2409_15097_b200/libbbm.so
timeout 900 bash abl_bin/run.sh
