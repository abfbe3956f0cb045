#!/bin/bash
# one ncu --set full capture of the attention kernel: CFG VARIANT TAG
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_fwd_kernel -s 3 -c 1 \
    -o gpurun_out/${3}_attn_$1_$2 -f python bench.py --profile --config $1 --variant $2 --steps 3 --warmup 3 > gpurun_out/${3}_ncu_$1_$2.log 2>&1
