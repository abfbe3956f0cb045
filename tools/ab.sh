#!/bin/bash
# A/B forward timing of in-tree builds (run under gpurun):
#   LIBS="prev pair" CONFIGS="c5:binblk c2:dense" bash tools/ab.sh
# lib "cur" = paper_2409_15097_b200/libbbm.so, any other name X = abl_bin/libbbm_X.so
mkdir -p gpurun_out
CONFIGS=${CONFIGS:-"c5:binblk c2:binblk c2:dense c4:dense-binblk c3:binblk"}
LIBS=${LIBS:-"prev cur"}
for spec in $CONFIGS; do
  cfg=${spec%%:*}; var=${spec##*:}
  for rep in ${REPS:-1 2 3}; do
  for lib in $LIBS; do
    if [ $lib = cur ]; then unset BBM_LIB; else export BBM_LIB=$PWD/abl_bin/libbbm_$lib.so; fi
    r=$(timeout 300 python bench.py --config $cfg --variant $var --steps 20 --warmup 5 ${ABPASS:+--pass $ABPASS} ${ABMODE:---profile} 2>&1 | tail -1)
    echo "$cfg $var $lib $r" | tee -a gpurun_out/ab.log
  done
  done
done
