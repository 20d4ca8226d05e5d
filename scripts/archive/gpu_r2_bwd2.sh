# bwd_row in fp32 pairs with the token entry stored after the loop; deferred pass without the
# finalize round trip. Full GPU suite, then same-box A/B against the previous commit's build
# (build/prev) on the two-call and deferred steps, then the deferred phase trace.
mkdir -p gpurun_out
timeout 1800 python -m pytest -q -m gpu tests -x 2>&1 | tail -3
for rep in 1 2; do
for v in prev prod; do
  if [ $v = prod ]; then L=""; else L="$PWD/build/prev/libtba.so"; fi
  for spec in qwen_shard:two-call rhomath:two-call pythia:two-call qwen_shard:deferred math_t5_shard:deferred pythia_fp32:deferred rhomath:deferred; do
    wl=${spec%%:*}; sch=${spec##*:}
    TBA_LIBRARY=$L timeout 300 python bench.py --workload $wl --schedule $sch --no-e2e --no-cpu-baseline --no-variants > gpurun_out/b2_${v}_${wl}_$sch.json 2>gpurun_out/b2_${v}_${wl}_$sch.err
    python -c "
import json; d=json.load(open('gpurun_out/b2_${v}_${wl}_$sch.json')); r=d['roofline']; print('$v', '$wl', '$sch', round(d['ms_per_step'],4), round(r['frac'],3), r.get('fwd_frac'), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/b2_${v}_${wl}_$sch.err
  done
done
done
python scripts/ab_variants.py trace=TBA_AB_DEFER_TRACE > /dev/null 2>&1
TBA_LIBRARY=/tmp/tba_variants/trace/libtba.so timeout 600 python scripts/defer_trace.py
