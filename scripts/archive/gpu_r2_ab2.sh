# A/B 2: uniform-iteration token exclusion vs none; SMEM-resident deferred pass vs the L2 two-pass
# kernel; hostile tests; an ncu --set full capture of row_smem on one Qwen group.
mkdir -p gpurun_out
python scripts/ab_variants.py noexcl=TBA_AB_NO_EXCL deferl2=TBA_AB_DEFER_L2 > /dev/null 2>&1
timeout 600 python -m pytest -q tests/test_gpu_hostile.py 2>&1 | grep -E "Error|passed|failed" | head -20
for rep in 1 2; do
for v in prod noexcl deferl2; do
  if [ $v = prod ]; then L=""; else L="/tmp/tba_variants/$v/libtba.so"; fi
  for wl in qwen_shard pythia gsm8k_t3; do
    TBA_LIBRARY=$L timeout 600 python bench.py --workload $wl --no-e2e --no-cpu-baseline > gpurun_out/ab2_${v}_$wl.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/ab2_${v}_$wl.json')); k=d['kernels']
print('$v', '$wl', round(d['ms_per_step'],4), 'fwd', round(k['fwd_ms'],4), 'bwd', round(k['bwd_ms'],4), 'defer', round(d['variants']['deferred_scale']['ms_per_step'],4), d['clocks']['sm_mhz'])"
  done
done
done
timeout 900 ncu --set full --clock-control none -k regex:row_smem -c 1 -o gpurun_out/ncu_row_smem_qwen_group \
  python bench.py --workload qwen_group --schedule deferred --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-variants > /dev/null 2>&1
ls -la gpurun_out/ncu_row_smem_qwen_group* 2>&1 | tail -1
