#!/bin/bash
# Split-unit sweep (BBM_MIN_UNIT) on the small configs, alternating values within one session.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/minunit
for rep in 1 2; do
  for mu in 16 8 4 2; do
    for cfg in "c1 binblk" "c1 dense" "c3 binblk" "c4 dense-binblk"; do
      set -- $cfg
      BBM_MIN_UNIT=$mu timeout 120 python bench.py --config $1 --variant $2 --steps 30 --warmup 5 --no-cpu-baseline \
        --no-e2e > gpurun_out/minunit/$1_$2_mu${mu}_r$rep.json 2>/dev/null
      python - "$1" "$2" "$mu" "$rep" <<'PY'
import json, sys
c, v, mu, rep = sys.argv[1:]
try:
    d = json.loads(open(f"gpurun_out/minunit/{c}_{v}_mu{mu}_r{rep}.json").read().strip().splitlines()[-1])
    print(f"{c} {v} mu={mu} r{rep}: {d['ms_per_step']*1000:.1f} us  kernel {d['roofline']['flops_per_launch']/d['roofline']['achieved']/1e6:.1f} us  {d['clocks']['sm_mhz']} MHz")
except Exception as e:
    print(c, v, mu, rep, "failed", e)
PY
    done
  done
done
