# A/B: stash size of the deferred kernel's long-row configuration (0 = the round-1 L2 kernel), same box.
mkdir -p gpurun_out
python scripts/ab_variants.py s0=TBA_DEFER_STASH_KB=0 s64=TBA_DEFER_STASH_KB=64 s104=TBA_DEFER_STASH_KB=104 s110=TBA_DEFER_STASH_KB=110 > /dev/null 2>&1
for rep in 1 2; do
for v in prod s0 s64 s104 s110; do
  if [ $v = prod ]; then L=""; else L="/tmp/tba_variants/$v/libtba.so"; fi
  for wl in qwen_shard pythia_fp32; do
    TBA_LIBRARY=$L timeout 300 python bench.py --workload $wl --schedule deferred --no-e2e --no-cpu-baseline --no-variants > gpurun_out/s2_${v}_$wl.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/s2_${v}_$wl.json')); print('$v', '$wl', round(d['ms_per_step'],4), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
  done
done
done
