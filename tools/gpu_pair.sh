#!/bin/bash
# pair-kernel bring-up: parity tests, then timings of both kernels and the fast-engine ablation
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 180 python -m pytest tests/test_gpu_pair.py -x -q > gpurun_out/p_test.log 2>&1; echo "rc=$?" >> gpurun_out/p_test.log
for k in single pair; do
 for spec in "c5 binblk" "c2 binblk" "c2 dense" "c3 binblk"; do set -- $spec
  BBM_FWD_KERNEL=$k timeout 150 python bench.py --config $1 --variant $2 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python tools/bench_summary.py | sed "s/^/$k /" >> gpurun_out/p_bench.txt
 done
done
if [ -f abl_bin/libbbm_FAST_ENGINE.so ]; then
  cp paper_2409_15097_b200/libbbm.so /tmp/libbbm_real.so
  cp abl_bin/libbbm_FAST_ENGINE.so paper_2409_15097_b200/libbbm.so
  for k in single pair; do
   for spec in "c5 binblk" "c2 dense"; do set -- $spec
    BBM_FWD_KERNEL=$k timeout 150 python bench.py --config $1 --variant $2 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python tools/bench_summary.py | sed "s/^/FAST $k /" >> gpurun_out/p_bench.txt
   done
  done
  cp /tmp/libbbm_real.so paper_2409_15097_b200/libbbm.so
fi
