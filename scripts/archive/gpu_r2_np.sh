# A/B: FMA-pipe exp2 offload (NP pairs of each vector) in the deferred passes 1 / 2 vs none (the product).
mkdir -p gpurun_out
python scripts/ab_variants.py np10=TBA_DEFER_NP1=1 np01=TBA_DEFER_NP2=1 np11=TBA_DEFER_NP1=1,TBA_DEFER_NP2=1 np21=TBA_DEFER_NP1=2,TBA_DEFER_NP2=1 np12=TBA_DEFER_NP1=1,TBA_DEFER_NP2=2 np22=TBA_DEFER_NP1=2,TBA_DEFER_NP2=2 > /dev/null 2>&1
for v in np11 np22; do
TBA_LIBRARY=/tmp/tba_variants/$v/libtba.so timeout 900 python -m pytest -q -m gpu tests/test_gpu_fused.py tests/test_gpu_tbap.py -k deferred 2>&1 | tail -1
done
for rep in 1 2; do
for v in prod np10 np01 np11 np21 np12 np22; do
  if [ $v = prod ]; then L=""; else L="/tmp/tba_variants/$v/libtba.so"; fi
  for wl in qwen_shard math_t5_shard rhomath pythia_fp32; do
    TBA_LIBRARY=$L timeout 300 python bench.py --workload $wl --schedule deferred --no-e2e --no-cpu-baseline --no-variants > gpurun_out/np_${v}_$wl.json 2>gpurun_out/np_${v}_$wl.err
    python -c "
import json; d=json.load(open('gpurun_out/np_${v}_$wl.json')); print('$v', '$wl', round(d['ms_per_step'],4), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/np_${v}_$wl.err
  done
done
done
