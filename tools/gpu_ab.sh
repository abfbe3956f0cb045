#!/bin/bash
# quick A/B: forward parity tests + bench lines of the main configs (run under gpurun)
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gpu_prep.py tests/test_gpu_attn.py tests/test_gpu_pair.py tests/test_gpu_fullsize.py tests/test_gpu_bwd.py -x -q > gpurun_out/ab_test.log 2>&1; echo "rc=$?" >> gpurun_out/ab_test.log
for rep in 1 2; do
for spec in "c5 binblk" "c2 binblk" "c2 dense" "c3 binblk" "c4 dense-binblk"; do set -- $spec
  timeout 150 python bench.py --config $1 --variant $2 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python tools/bench_summary.py >> gpurun_out/ab_bench.txt
done
done
