# A/B: the deferred-scale kernel's configuration (TBA_AB_DEFER_CFG: 1 = 8 vectors per thread in pass 1,
# 2 = 1024 threads per row) against the product (512 threads, 4 / 8 vectors), same box, interleaved.
mkdir -p gpurun_out
python scripts/ab_variants.py dcfg1=TBA_AB_DEFER_CFG=1 dcfg2=TBA_AB_DEFER_CFG=2 > /dev/null 2>&1
for rep in 1 2; do
for v in prod dcfg1 dcfg2; do
  if [ $v = prod ]; then L=""; else L="/tmp/tba_variants/$v/libtba.so"; fi
  for wl in qwen_shard rhomath pythia; do
    TBA_LIBRARY=$L timeout 300 python bench.py --workload $wl --schedule deferred --no-e2e --no-cpu-baseline --no-variants > gpurun_out/df_${v}_$wl.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/df_${v}_$wl.json')); print('$v', '$wl', round(d['ms_per_step'],4), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
  done
done
done
L=/tmp/tba_variants/dcfg2/libtba.so
TBA_LIBRARY=$L ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:row_single -s 3 -c 1 --csv python bench.py --workload qwen_shard --schedule deferred --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-variants 2>/dev/null | grep -E "dram|duration" | cut -d, -f12- | head
