# A/B: the deferred pass with the row kept on chip across a cluster (row_slab, TBA_AB_SLAB) vs the
# product (row_single1: L2 re-read + 96 KB cp.async stash); parity of the variants first.
mkdir -p gpurun_out
python scripts/ab_variants.py slab=TBA_AB_SLAB slab4=TBA_AB_SLAB,TBA_SLAB_U=4 slab256=TBA_AB_SLAB,TBA_SLAB_NT=256,TBA_SLAB_CAP_KB=50 > gpurun_out/slab_build.log 2>&1
for v in slab slab256; do
TBA_LIBRARY=/tmp/tba_variants/$v/libtba.so timeout 900 python -m pytest -q -m gpu tests/test_gpu_fused.py tests/test_gpu_tbap.py -k deferred 2>&1 | tail -3
done
for rep in 1 2; do
for v in prod slab slab4 slab256; do
  if [ $v = prod ]; then L=""; else L="/tmp/tba_variants/$v/libtba.so"; fi
  for wl in qwen_shard math_t5_shard pythia pythia_fp32 rhomath; do
    TBA_LIBRARY=$L timeout 300 python bench.py --workload $wl --schedule deferred --no-e2e --no-cpu-baseline --no-variants > gpurun_out/sl_${v}_$wl.json 2>gpurun_out/sl_${v}_$wl.err
    python -c "
import json; d=json.load(open('gpurun_out/sl_${v}_$wl.json')); print('$v', '$wl', round(d['ms_per_step'],4), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/sl_${v}_$wl.err
  done
done
done
