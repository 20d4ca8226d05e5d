# A/B: the deferred kernel keeping the row's first 64 / 96 KB in shared memory between its passes
# (TBA_AB_DEFER_STASH) against the product, same box, interleaved; DRAM bytes of the best.
mkdir -p gpurun_out
python scripts/ab_variants.py st96=TBA_AB_DEFER_STASH=96 st96c3=TBA_AB_DEFER_STASH=96,TBA_AB_DEFER_CFG=3 st64c3=TBA_AB_DEFER_STASH=64,TBA_AB_DEFER_CFG=3 > /dev/null 2>&1
timeout 600 env TBA_LIBRARY=/tmp/tba_variants/st96c3/libtba.so python -m pytest -q -m gpu tests/test_gpu_fused.py -k deferred 2>&1 | tail -1
for rep in 1 2; do
for v in prod st96 st96c3 st64c3; do
  if [ $v = prod ]; then L=""; else L="/tmp/tba_variants/$v/libtba.so"; fi
  for wl in qwen_shard rhomath pythia redteam; do
    TBA_LIBRARY=$L timeout 300 python bench.py --workload $wl --schedule deferred --no-e2e --no-cpu-baseline --no-variants > gpurun_out/st_${v}_$wl.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/st_${v}_$wl.json')); print('$v', '$wl', round(d['ms_per_step'],4), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
  done
done
done
for v in st96c3 st64c3; do
TBA_LIBRARY=/tmp/tba_variants/$v/libtba.so ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:row_single -s 3 -c 1 --csv python bench.py --workload qwen_shard --schedule deferred --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-variants 2>/dev/null | grep -E "dram|duration" | awk -F'","' '{print "'$v'", $(NF-2), $NF}'
done
