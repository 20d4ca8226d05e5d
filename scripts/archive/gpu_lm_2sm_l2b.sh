# 2-SM LM head: raster super-row size (in SM-pair units) vs DRAM bytes and time.
B="python bench.py --objective lmhead --no-e2e --no-cpu-baseline --no-variants --steps 1 --warmup 3"
for swz in 16 8 4; do
  TBA_LM_MC=3 TBA_LM_POL=5 TBA_LM_SWZ=$swz timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:lmhead_fwd -s 3 -c 1 --csv $B 2>/dev/null | grep -E "dram__bytes_read|hit_rate|duration" | awk -F'","' -v t="mc=3 swz=$swz" '{print t, $(NF-2), $NF}'
done
for swz in 32 16; do
  TBA_LM_MC=1 TBA_LM_SWZ=$swz timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:lmhead_fwd -s 3 -c 1 --csv $B 2>/dev/null | grep -E "dram__bytes_read|hit_rate|duration" | awk -F'","' -v t="mc=1 swz=$swz" '{print t, $(NF-2), $NF}'
done
run() {
  env "$@" timeout 300 python bench.py --objective lmhead --steps 8 --warmup 3 --no-e2e --no-cpu-baseline \
    --no-variants 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('%-44s ms=%.2f  TF/s=%.0f  sm_mhz=%s' % ('$*', d['ms_per_step'], d['roofline']['achieved'], d['clocks']['sm_mhz']))"
}
for rep in 1 2; do
run TBA_LM_MC=3 TBA_LM_POL=5 TBA_LM_SWZ=8
run TBA_LM_MC=3 TBA_LM_POL=5 TBA_LM_SWZ=4
run TBA_LM_MC=1
done
