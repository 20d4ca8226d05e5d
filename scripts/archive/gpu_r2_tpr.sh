# A/B: forward with one warp per row for rows < N vectors (t32: 128 KB rows, + NP=1 offload t32np)
mkdir -p gpurun_out
python scripts/ab_variants.py t32=TBA_FWD_TPR32_BELOW=8192 t32np=TBA_FWD_TPR32_BELOW=8192,TBA_FWD_NP32=1 > /dev/null 2>&1
TBA_LIBRARY=/tmp/tba_variants/t32np/libtba.so timeout 900 python -m pytest -q -m gpu tests/test_gpu_parity.py 2>&1 | tail -1
B="python bench.py --no-e2e --no-cpu-baseline --no-variants"
for rep in 1 2; do
for v in prod t32 t32np; do
  if [ $v = prod ]; then L=""; else L="/tmp/tba_variants/$v/libtba.so"; fi
  for wl in pythia redteam gsm8k_t3 gsm8k_k40 rhomath; do
  TBA_LIBRARY=$L $B --workload $wl > gpurun_out/tp_${v}_$wl.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/tp_${v}_$wl.json')); k=d['kernels']; print('$v', '$wl', round(d['ms_per_step'],4), 'fwd', round(k['fwd_ms'],4), round(k['fwd_frac'],3), 'bwd', round(k['bwd_ms'],4), 'step', round(k['step_frac'],3), d['clocks']['sm_mhz'])"
  done
done
done
