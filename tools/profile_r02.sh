#!/bin/bash
# Round-2 ncu evidence (run under gpurun, one GPU):
#  - the launch list of the default bench (C5) with per-launch device times
#  - one --set full capture of the forward kernel (C5 binblk, C2 dense) and of the fused preprocessor (C5, C2)
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/r02_launches_c5.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline \
  > gpurun_out/r02_launches_c5.log 2>&1
for spec in "c5 binblk" "c2 dense"; do set -- $spec
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd_kernel -s 3 -c 1 \
    -o gpurun_out/r02_attn_$1_$2 -f python bench.py --profile --config $1 --variant $2 --steps 3 --warmup 3 \
    > gpurun_out/r02_ncu_attn_$1_$2.log 2>&1
done
for c in c5 c2; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:prep_fused -s 2 -c 1 \
    -o gpurun_out/r02_prep_$c -f python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline \
    > gpurun_out/r02_ncu_prep_$c.log 2>&1
done
ls -la gpurun_out/
