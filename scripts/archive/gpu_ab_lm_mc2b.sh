# LM head: multicast pair (raster in row blocks) vs single-CTA, interleaved, each paired with cuBLAS.
run() {
  env "$@" timeout 300 python bench.py --objective lmhead --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); u=d['variants']['unfused_cublas_logits']
print('%-14s fused %.2f ms (%s MHz)  paired fused %.2f unfused %.2f ratio %.3f' % ('$*', d['ms_per_step'], d['clocks']['sm_mhz'], u['fused_ms_paired'], u['ms_per_step'], u['fused_over_unfused']))"
}
for rep in 1 2 3; do run TBA_LM_MC=1; run TBA_LM_MC=2; done
B="python bench.py --objective lmhead --no-e2e --no-cpu-baseline --no-variants --steps 1 --warmup 3"
for mc in 1 2; do TBA_LM_MC=$mc timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:lmhead_fwd -s 3 -c 1 --csv $B 2>/dev/null | grep -E "dram__bytes_read|duration" | awk -F'","' -v t="mc=$mc" '{print t, $(NF-2), $NF}'; done
