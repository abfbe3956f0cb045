nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for c in c1 c2 c3 c4 c5; do
 v=binblk; [ $c = c4 ] && v=dense-binblk
 timeout 300 python bench.py --config $c --variant $v --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1
done
timeout 300 python bench.py > gpurun_out/bench_default.log 2>&1
