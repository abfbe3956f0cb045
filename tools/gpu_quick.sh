#!/bin/bash
# quick loop: forward parity + C2/C4/C5 bench lines + traces (run under gpurun)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_attn.py tests/test_gpu_bwd.py -x -q > gpurun_out/q_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/q_pytest.log
for spec in "c2 binblk" "c2 dense" "c4 dense-binblk" "c5 binblk" "c3 binblk"; do set -- $spec
  timeout 300 python bench.py --config $1 --variant $2 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python tools/bench_summary.py >> gpurun_out/q_bench.txt
done
for spec in "c2 dense" "c2 binblk" "c4 dense-binblk"; do set -- $spec
  timeout 120 python tools/trace_attn.py --config $1 --variant $2 --ctas 1 > gpurun_out/q_trace_$1_$2.txt 2>&1
done
