#!/bin/bash
# ncu evidence for profiles/: a launch list of the bench command and one --set full capture of
# the attention kernel per config, plus the preprocessor's bool-pack kernel. Run under gpurun.
set -x
mkdir -p gpurun_out
TAG=${TAG:-r01}
ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv \
    --log-file gpurun_out/${TAG}_launches_c2.csv python bench.py --profile --steps 5 --warmup 3 > /dev/null 2>&1
for spec in "c2 binblk" "c2 dense" "c4 dense-binblk" "c5 binblk" "c3 binblk"; do
  set -- $spec
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_fwd_kernel -s 3 -c 1 \
      -o gpurun_out/${TAG}_attn_$1_$2 -f python bench.py --profile --config $1 --variant $2 --steps 3 --warmup 3 > gpurun_out/${TAG}_ncu_$1_$2.log 2>&1
done
timeout 600 ncu --set full --clock-control none -k regex:pack_bool -c 1 -o gpurun_out/${TAG}_prep_c5 -f \
    python bench.py --profile --config c5 --steps 3 --warmup 3 > gpurun_out/${TAG}_ncu_prep.log 2>&1
ls -la gpurun_out
