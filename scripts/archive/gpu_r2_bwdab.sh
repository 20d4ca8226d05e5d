# A/B of the bwd_row loop: pairs vs scalar arithmetic, token entry in the loop vs after it
mkdir -p gpurun_out
python scripts/ab_variants.py scalar=TBA_AB_BWD_SCALAR inloop=TBA_AB_BWD_TOK_INLOOP both=TBA_AB_BWD_SCALAR,TBA_AB_BWD_TOK_INLOOP > /dev/null 2>&1
for rep in 1 2; do
for v in prev prod scalar inloop both; do
  if [ $v = prod ]; then L=""; elif [ $v = prev ]; then L="$PWD/build/prev/libtba.so"; else L="/tmp/tba_variants/$v/libtba.so"; fi
  for spec in qwen_shard:two-call pythia:two-call qwen_shard:deferred; do
    wl=${spec%%:*}; sch=${spec##*:}
    TBA_LIBRARY=$L timeout 300 python bench.py --workload $wl --schedule $sch --no-e2e --no-cpu-baseline --no-variants > gpurun_out/ba_${v}_${wl}_$sch.json 2>gpurun_out/ba_${v}_${wl}_$sch.err
    python -c "
import json; d=json.load(open('gpurun_out/ba_${v}_${wl}_$sch.json')); r=d['roofline']; print('$v', '$wl', '$sch', round(d['ms_per_step'],4), round(r['frac'],3), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/ba_${v}_${wl}_$sch.err
  done
done
done
