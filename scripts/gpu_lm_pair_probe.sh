# Pair-schedule L2 probe: multicast vs per-CTA weight loads in the cluster pair, vs the single-CTA kernel.
B="python bench.py --objective lmhead --no-e2e --no-cpu-baseline --no-variants --steps 1 --warmup 3"
for cfg in "TBA_LM_MC=2 TBA_LM_POL=1" "TBA_LM_MC=2 TBA_LM_POL=9" "TBA_LM_MC=2 TBA_LM_POL=9 TBA_LM_SWZ=16" "TBA_LM_MC=1 TBA_LM_POL=1"; do
  env $cfg timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:lmhead_fwd -s 3 -c 1 --csv $B 2>/dev/null | grep -E "dram__bytes_read|hit_rate|duration" | awk -F'","' -v t="$cfg" '{print t, $(NF-2), $NF}'
done
