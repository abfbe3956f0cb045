#!/bin/bash
# event traces of the forward kernel for a few configs (run under gpurun)
mkdir -p gpurun_out
for spec in ${SPECS:-"c2 dense" "c2 binblk" "c4 dense-binblk" "c5 binblk"}; do set -- $spec
  timeout 120 python tools/trace_attn.py --config $1 --variant $2 --ctas 2 > gpurun_out/t_trace_$1_$2.txt 2>&1
done
