B="python bench.py --objective lmhead --no-e2e --no-cpu-baseline --no-variants --steps 1 --warmup 3"
for mc in 2 3 1; do
  TBA_LM_MC=$mc timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none -k regex:lmhead_fwd -s 3 -c 1 --csv $B 2>/dev/null | grep -E "dram__bytes_read|hit_rate|duration|srcunit" | awk -F'","' -v t="mc=$mc" '{print t, $(NF-2), $NF}'
done
