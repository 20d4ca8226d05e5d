# A/B: L2 bulk prefetch of the whole row up front in the deferred pass for rows <= 128 KB
mkdir -p gpurun_out
python scripts/ab_variants.py pfs=TBA_AB_DEFER_PF_SMALL > /dev/null 2>&1
TBA_LIBRARY=/tmp/tba_variants/pfs/libtba.so timeout 900 python -m pytest -q -m gpu tests/test_gpu_fused.py tests/test_gpu_tbap.py -k deferred 2>&1 | tail -1
for rep in 1 2; do
for v in prod pfs; do
  if [ $v = prod ]; then L=""; else L="/tmp/tba_variants/$v/libtba.so"; fi
  for wl in rhomath pythia redteam qwen_shard; do
    TBA_LIBRARY=$L timeout 300 python bench.py --workload $wl --schedule deferred --no-e2e --no-cpu-baseline --no-variants > gpurun_out/ps_${v}_$wl.json 2>gpurun_out/ps_${v}_$wl.err
    python -c "
import json; d=json.load(open('gpurun_out/ps_${v}_$wl.json')); print('$v', '$wl', round(d['ms_per_step'],4), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/ps_${v}_$wl.err
  done
done
done
