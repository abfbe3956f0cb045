# instructions executed / duration of the forward kernel per lib (A/B sanity, not a bench number)
mkdir -p gpurun_out
for cfg in ${CONFIGS:-"c5:binblk"}; do c=${cfg%%:*}; v=${cfg##*:}
for lib in $LIBS; do
  BBM_LIB=$PWD/abl_bin/libbbm_$lib.so timeout 600 ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:attn_fwd_kernel -s 3 -c 1 --csv \
    python bench.py --profile --config $c --variant $v --steps 3 --warmup 3 2>/dev/null | grep -E '"(smsp|gpu__|sm__)' | awk -F'","' -v l=$lib -v c=$c '{print c, l, $(NF-2), $NF}'
done; done
