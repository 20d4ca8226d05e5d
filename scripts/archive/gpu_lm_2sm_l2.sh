# 2-SM LM head: is the L2 miss storm tied to the TMA cache hint? DRAM bytes + time per variant.
B="python bench.py --objective lmhead --no-e2e --no-cpu-baseline --no-variants --steps 1 --warmup 3"
for pol in 1 5 4; do
  TBA_LM_MC=3 TBA_LM_POL=$pol timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:lmhead_fwd -s 3 -c 1 --csv $B 2>/dev/null | grep -E "dram__bytes_read|hit_rate|duration" | awk -F'","' -v t="mc=3 pol=$pol" '{print t, $(NF-2), $NF}'
done
run() {
  env "$@" timeout 300 python bench.py --objective lmhead --steps 8 --warmup 3 --no-e2e --no-cpu-baseline \
    --no-variants 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('%-36s ms=%.2f  TF/s=%.0f  sm_mhz=%s' % ('$*', d['ms_per_step'], d['roofline']['achieved'], d['clocks']['sm_mhz']))"
}
run TBA_LM_MC=3 TBA_LM_POL=5
run TBA_LM_MC=1
run TBA_LM_MC=3 TBA_LM_POL=5
run TBA_LM_MC=1
