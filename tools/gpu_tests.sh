#!/bin/bash
# GPU parity suite + C++ drop-in + a traced forward (run under gpurun)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for spec in "c2 dense" "c2 binblk"; do set -- $spec
  timeout 120 python tools/trace_attn.py --config $1 --variant $2 --ctas 2 > gpurun_out/trace_$1_$2.txt 2>&1
done
