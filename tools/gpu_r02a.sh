#!/bin/bash
# round-2 checkpoint run (under gpurun, one GPU): full GPU suite, smoke, default bench (C5 with
# CPU baseline + e2e), the reference arm, per-config forward / backward lines, C5 launch list
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/smi.txt 2>&1
lscpu > gpurun_out/lscpu.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.log 2>&1
for spec in "c1 binblk" "c2 binblk" "c2 dense" "c3 binblk" "c4 dense-binblk" "c4 dense" "c5 dense"; do set -- $spec
  timeout 300 python bench.py --config $1 --variant $2 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_$1_$2.log 2>&1
done
for spec in "c2 binblk" "c4 dense-binblk" "c5 binblk"; do set -- $spec
  timeout 300 python bench.py --pass bwd --config $1 --variant $2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_bwd_$1.log 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/r02_launches_c5.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline \
  > gpurun_out/r02_launches_c5.log 2>&1
ls -la gpurun_out/
