# 2-SM probe: stage completions relayed through the peer (plain TMA) vs .cta_group::2 loads.
TBA_LM_MC=3 TBA_LM_POL=17 TBA_LM_SWZ=16 timeout 120 python scripts/lmhead_debug.py 2>&1 | tail -3
TBA_LM_MC=3 TBA_LM_POL=17 TBA_LM_SWZ=16 timeout 300 python -m pytest tests/test_gpu_lmhead.py -q -x -k "lattice or tb_head" 2>&1 | tail -1
B="python bench.py --objective lmhead --no-e2e --no-cpu-baseline --no-variants --steps 1 --warmup 3"
for cfg in "TBA_LM_MC=3 TBA_LM_POL=17 TBA_LM_SWZ=16" "TBA_LM_MC=3 TBA_LM_POL=17 TBA_LM_SWZ=8" "TBA_LM_MC=3 TBA_LM_POL=1 TBA_LM_SWZ=16"; do
  env $cfg timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:lmhead_fwd -s 3 -c 1 --csv $B 2>/dev/null | grep -E "dram__bytes_read|hit_rate|duration" | awk -F'","' -v t="$cfg" '{print t, $(NF-2), $NF}'
done
run() {
  env "$@" timeout 300 python bench.py --objective lmhead --steps 8 --warmup 3 --no-e2e --no-cpu-baseline \
    --no-variants 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('%-44s ms=%.2f  TF/s=%.0f  sm_mhz=%s' % ('$*', d['ms_per_step'], d['roofline']['achieved'], d['clocks']['sm_mhz']))"
}
for rep in 1 2; do run TBA_LM_MC=3 TBA_LM_POL=17 TBA_LM_SWZ=16; run TBA_LM_MC=1; done
