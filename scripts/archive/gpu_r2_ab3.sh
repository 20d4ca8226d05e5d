# A/B 3: SMEM-resident deferred pass (16 KB tiles, 2 vectors per thread) vs the L2 kernel; hostile
# and deferred tests; ncu of row_smem on one Qwen group.
mkdir -p gpurun_out
python scripts/ab_variants.py deferl2=TBA_AB_DEFER_L2 > /dev/null 2>&1
timeout 600 python -m pytest -q tests/test_gpu_hostile.py 2>&1 | grep -E "Error|passed|failed" | head -20
timeout 900 python -m pytest -q tests/test_gpu_fused.py tests/test_gpu_tbap.py -k "deferred" 2>&1 | tail -2
for rep in 1 2; do
for v in prod deferl2; do
  if [ $v = prod ]; then L=""; else L="/tmp/tba_variants/$v/libtba.so"; fi
  for wl in qwen_shard pythia rhomath redteam; do
    TBA_LIBRARY=$L timeout 600 python bench.py --workload $wl --no-e2e --no-cpu-baseline > gpurun_out/ab3_${v}_$wl.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/ab3_${v}_$wl.json')); k=d['kernels']
print('$v', '$wl', round(d['ms_per_step'],4), 'fwd', round(k['fwd_ms'],4), 'bwd', round(k['bwd_ms'],4), 'defer', round(d['variants']['deferred_scale']['ms_per_step'],4), d['clocks']['sm_mhz'])"
  done
done
done
timeout 900 ncu --set full --clock-control none -k regex:row_smem -c 1 -o gpurun_out/ncu_row_smem2_qwen_group \
  python bench.py --workload qwen_group --schedule deferred --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-variants > /dev/null 2>&1
