#!/bin/bash
set -e
cp paper_2409_15097_b200/libbbm.so /tmp/libbbm_real.so
for v in NO_MUFU NO_XCHG; do
  cp ablate/libbbm_$v.so paper_2409_15097_b200/libbbm.so
  for var in binblk dense; do
    echo -n "$v "; python bench.py --config c2 --variant $var --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python3 tools/bench_summary.py
  done
done
cp /tmp/libbbm_real.so paper_2409_15097_b200/libbbm.so
