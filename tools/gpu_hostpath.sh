#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_prep_contract.py -x -q > gpurun_out/hp_test.log 2>&1; echo "rc=$?" >> gpurun_out/hp_test.log
for f in 0.7; do
  BBM_HOST_CONVERT=$f timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/hp_bench_$f.log 2>&1
done
