#!/bin/bash
# round-end evidence: full GPU suite, bench lines for every config (fwd + bwd), default bench with
# the CPU baseline, ncu launch list + full captures (run under gpurun)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for c in c1 c2 c3 c4 c5; do
 v=binblk; [ $c = c4 ] && v=dense-binblk
 timeout 300 python bench.py --config $c --variant $v --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1
 timeout 300 python bench.py --pass bwd --config $c --variant $v --steps 10 --warmup 3 > gpurun_out/bench_bwd_$c.log 2>&1
done
timeout 600 python bench.py > gpurun_out/bench_default.log 2>&1
TAG=${TAG:-r01} bash tools/profile.sh > gpurun_out/profile.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_bwd_kernel -s 2 -c 2 \
    -o gpurun_out/${TAG:-r01}_bwd_c2_binblk -f python bench.py --pass bwd --profile --config c2 --steps 2 --warmup 3 > gpurun_out/ncu_bwd.log 2>&1
