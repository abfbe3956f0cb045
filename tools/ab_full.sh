#!/bin/bash
# A/B of in-tree builds under the FULL bench protocol (soak + timed region, power-capped steady
# state), extracting value / ms / clocks:  LIBS="base suspend" CONFIGS="c5:binblk" bash tools/ab_full.sh
mkdir -p gpurun_out
CONFIGS=${CONFIGS:-"c5:binblk c2:binblk"}
LIBS=${LIBS:-"base cur"}
for spec in $CONFIGS; do
  cfg=${spec%%:*}; var=${spec##*:}
  for rep in 1 2; do
  for lib in $LIBS; do
    if [ $lib = cur ]; then unset BBM_LIB; else export BBM_LIB=$PWD/abl_bin/libbbm_$lib.so; fi
    r=$(timeout 300 python bench.py --config $cfg --variant $var --steps 20 --warmup 5 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), round(d['value'],1), d['clocks']['sm_mhz'], d['roofline']['avg_launch_ms'], d.get('dense_mask_run',{}).get('ms_per_step'))")
    echo "$cfg $var $lib $r" | tee -a gpurun_out/ab_full.log
  done
  done
done
