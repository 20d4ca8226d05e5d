# A/B: PDL on/off, PDL trigger, token exclusion, on the default bench line and the small shapes;
# then the hostile/deferred tests with full failure output.
mkdir -p gpurun_out
python scripts/ab_variants.py nopdl=TBA_AB_NO_PDL noexcl=TBA_AB_NO_EXCL notrig=TBA_AB_NO_PDL_TRIGGER > /dev/null 2>&1
timeout 600 python -m pytest -q -x tests/test_gpu_hostile.py 2>&1 | grep -E "Error|assert|passed|failed" | head -20
timeout 900 python -m pytest -q tests/test_gpu_fused.py tests/test_gpu_tbap.py -k "deferred" 2>&1 | tail -3
for rep in 1 2; do
for v in prod nopdl noexcl notrig; do
  if [ $v = prod ]; then L=""; else L="/tmp/tba_variants/$v/libtba.so"; fi
  for wl in qwen_shard pythia gsm8k_t3; do
    TBA_LIBRARY=$L timeout 600 python bench.py --workload $wl --no-e2e --no-cpu-baseline > gpurun_out/ab_${v}_$wl.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/ab_${v}_$wl.json')); k=d['kernels']
print('$v', '$wl', round(d['ms_per_step'],4), 'fwd', round(k['fwd_ms'],4), 'bwd', round(k['bwd_ms'],4), 'defer', round(d['variants']['deferred_scale']['ms_per_step'],4), d['clocks']['sm_mhz'])"
  done
done
done
