# A/B: deferred pass for rows <= 128 KB with the forward-order pass 2 loop (smallp2) vs bwd_row swept from the end
mkdir -p gpurun_out
python scripts/ab_variants.py smallp2=TBA_AB_SMALL_P2 > /dev/null 2>&1
TBA_LIBRARY=/tmp/tba_variants/smallp2/libtba.so timeout 900 python -m pytest -q -m gpu tests/test_gpu_fused.py tests/test_gpu_tbap.py tests/test_gpu_hostile.py -k "deferred or confident" 2>&1 | tail -1
B="python bench.py --no-e2e --no-cpu-baseline --no-variants --schedule deferred"
for rep in 1 2; do
for v in prod smallp2; do
  if [ $v = prod ]; then L=""; else L="/tmp/tba_variants/$v/libtba.so"; fi
  for wl in pythia redteam rhomath gsm8k_t3; do
  TBA_LIBRARY=$L $B --workload $wl > gpurun_out/sp2_${v}_$wl.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/sp2_${v}_$wl.json')); print('$v', '$wl', round(d['ms_per_step'],4), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
  done
done
done
