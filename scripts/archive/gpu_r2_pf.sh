# A/B: deferred pass 1 with an L2 bulk prefetch of the row's register part (whole rest up front, or
# N KB ahead of the loop) vs none (the product); then the phase trace of the best guess.
mkdir -p gpurun_out
python scripts/ab_variants.py pfall=TBA_DEFER_PF_KB=-1 pf64=TBA_DEFER_PF_KB=64 pf128=TBA_DEFER_PF_KB=128 pf32=TBA_DEFER_PF_KB=32 tracepf=TBA_AB_DEFER_TRACE,TBA_DEFER_PF_KB=-1 > /dev/null 2>&1
TBA_LIBRARY=/tmp/tba_variants/pfall/libtba.so timeout 900 python -m pytest -q -m gpu tests/test_gpu_fused.py tests/test_gpu_tbap.py -k deferred 2>&1 | tail -1
for rep in 1 2; do
for v in prod pfall pf32 pf64 pf128; do
  if [ $v = prod ]; then L=""; else L="/tmp/tba_variants/$v/libtba.so"; fi
  for wl in qwen_shard math_t5_shard pythia_fp32; do
    TBA_LIBRARY=$L timeout 300 python bench.py --workload $wl --schedule deferred --no-e2e --no-cpu-baseline --no-variants > gpurun_out/pf_${v}_$wl.json 2>gpurun_out/pf_${v}_$wl.err
    python -c "
import json; d=json.load(open('gpurun_out/pf_${v}_$wl.json')); print('$v', '$wl', round(d['ms_per_step'],4), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/pf_${v}_$wl.err
  done
done
done
TBA_LIBRARY=/tmp/tba_variants/tracepf/libtba.so timeout 600 python scripts/defer_trace.py
