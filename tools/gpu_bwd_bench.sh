#!/bin/bash
mkdir -p gpurun_out
for spec in "c2 binblk" "c2 dense" "c4 dense-binblk" "c3 binblk" "c5 binblk"; do set -- $spec
  echo -n "bwd "; timeout 300 python bench.py --pass bwd --config $1 --variant $2 --steps 10 --warmup 3 2>&1 | tail -1 | python tools/bench_summary.py
done > gpurun_out/bwd_bench.txt 2>&1
