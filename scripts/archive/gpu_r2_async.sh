# A/B: the deferred kernel's stash part fetched with cp.async (all in flight at once) vs loaded
# through registers (the product), same box, interleaved; parity of the variant first.
mkdir -p gpurun_out
python scripts/ab_variants.py async=TBA_AB_DEFER_ASYNC async64=TBA_AB_DEFER_ASYNC,TBA_DEFER_STASH_KB=64 > /dev/null 2>&1
TBA_LIBRARY=/tmp/tba_variants/async/libtba.so timeout 600 python -m pytest -q -m gpu tests/test_gpu_fused.py tests/test_gpu_tbap.py -k deferred 2>&1 | tail -1
for rep in 1 2; do
for v in prod async async64; do
  if [ $v = prod ]; then L=""; else L="/tmp/tba_variants/$v/libtba.so"; fi
  for wl in qwen_shard pythia_fp32 math_t5_shard; do
    TBA_LIBRARY=$L timeout 300 python bench.py --workload $wl --schedule deferred --no-e2e --no-cpu-baseline --no-variants > gpurun_out/as_${v}_$wl.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/as_${v}_$wl.json')); print('$v', '$wl', round(d['ms_per_step'],4), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
  done
done
done
