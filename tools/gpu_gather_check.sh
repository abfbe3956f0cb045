mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_attn.py -q -x -k "gather" > gpurun_out/c_gather_test.log 2>&1; echo rc=$? >> gpurun_out/c_gather_test.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c_bench_c5.log 2>&1
