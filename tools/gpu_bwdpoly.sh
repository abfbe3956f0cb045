#!/bin/bash
# backward exp2 polynomial offload: parity + bwd timings of the base build and variants
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 400 python -m pytest tests/test_gpu_bwd.py -x -q > gpurun_out/bp_test.log 2>&1; echo "rc=$?" >> gpurun_out/bp_test.log
cp paper_2409_15097_b200/libbbm.so /tmp/libbbm_real.so
for v in base BWD_POLY0 BWD_POLY8 BWD_POLY10; do
  if [ $v = base ]; then cp /tmp/libbbm_real.so paper_2409_15097_b200/libbbm.so; else cp abl_bin/libbbm_$v.so paper_2409_15097_b200/libbbm.so; fi
  for spec in "c4 dense-binblk" "c2 binblk" "c5 binblk"; do set -- $spec
    echo -n "$v "; timeout 150 python bench.py --pass bwd --config $1 --variant $2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python3 tools/bench_summary.py
  done
done > gpurun_out/bp_bench.txt 2>&1
cp /tmp/libbbm_real.so paper_2409_15097_b200/libbbm.so
