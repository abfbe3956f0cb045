#!/bin/bash
# round-2 final evidence (one GPU): full GPU suite, smoke, default bench (C5 + CPU baseline + e2e),
# the reference arm, per-config fwd / bwd lines, the default bench's launch list, ncu --set full of
# the C5 forward and the C5 / C2 preprocessor, the C2 dense forward
mkdir -p gpurun_out/final
export PYTHONUNBUFFERED=1
O=gpurun_out/final
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/smi.txt 2>&1
lscpu > $O/lscpu.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_default.log 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.log 2>&1
for spec in "c1 binblk" "c2 binblk" "c2 dense" "c3 binblk" "c4 dense-binblk" "c4 dense" "c5 dense"; do set -- $spec
  timeout 300 python bench.py --config $1 --variant $2 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/bench_$1_$2.log 2>&1
done
for spec in "c2 binblk" "c4 dense-binblk" "c5 binblk"; do set -- $spec
  timeout 300 python bench.py --pass bwd --config $1 --variant $2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_bwd_$1.log 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/r02_launches_c5.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline \
  > $O/r02_launches_c5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd_kernel -s 3 -c 1 \
  -o $O/r02_attn_c5_binblk -f python bench.py --profile --config c5 --variant binblk --steps 3 --warmup 3 \
  > $O/ncu_attn_c5.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_bwd_kernel -s 2 -c 2 \
  -o $O/r02_bwd_c4 -f python bench.py --pass bwd --profile --config c4 --variant dense-binblk --steps 2 --warmup 3 \
  > $O/ncu_bwd_c4.log 2>&1
ls -la $O
