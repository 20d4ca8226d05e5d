# LM head: L2 policy bits (TBA_LM_POL: 1 weight evict_last, 2 hidden evict_last) x kernel variant.
run() {
  env "$@" timeout 300 python bench.py --objective lmhead --steps 8 --warmup 3 --no-e2e --no-cpu-baseline \
    --no-variants 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('%-36s ms=%.2f  TF/s=%.0f  sm_mhz=%s' % ('$*', d['ms_per_step'], d['roofline']['achieved'], d['clocks']['sm_mhz']))"
}
for rep in 1 2; do
  for pol in 1 0 2 3; do run TBA_LM_MC=1 TBA_LM_POL=$pol; done
  for pol in 1 0 2 3; do run TBA_LM_MC=3 TBA_LM_POL=$pol; done
done
B="python bench.py --objective lmhead --no-e2e --no-cpu-baseline --no-variants --steps 1 --warmup 3"
for mc in 1 3; do for pol in 0 1 2; do
  TBA_LM_MC=$mc TBA_LM_POL=$pol timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:lmhead_fwd -s 3 -c 1 --csv $B 2>/dev/null | grep -E "dram__bytes_read|hit_rate" | awk -F'","' -v t="mc=$mc pol=$pol" '{print t, $(NF-2), $NF}'
done; done
