#!/bin/bash
# timing-only ablations (results numerically wrong by design)
set -e
cp paper_2409_15097_b200/libbbm.so /tmp/libbbm_real.so
for v in nomufu noxchg; do
  cp ablate/libbbm_$v.so paper_2409_15097_b200/libbbm.so
  echo "== $v"; python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python3 tools/bench_summary.py
  python bench.py --config c2 --variant dense --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python3 tools/bench_summary.py
done
cp /tmp/libbbm_real.so paper_2409_15097_b200/libbbm.so
echo "== real"; python bench.py --config c2 --variant dense --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python3 tools/bench_summary.py
