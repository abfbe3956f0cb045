#!/bin/bash
mkdir -p gpurun_out/final
O=gpurun_out/final
timeout 900 python bench.py > $O/bench_default.log 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.log 2>&1
timeout 600 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
