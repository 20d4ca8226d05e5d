# Forward on the smaller-vocabulary shapes: rows-per-CTA LDG kernel (default) vs the persistent TMA ring.
B="python bench.py --no-e2e --no-cpu-baseline --no-variants --steps 30 --warmup 5"
for rep in 1 2; do
for w in pythia redteam gsm8k_t3 rhomath; do
  for cfg in "" "TBA_FWD_IMPL=tma TBA_TMA_CFG=3" "TBA_FWD_IMPL=tma TBA_TMA_CFG=0" "TBA_FWD_IMPL=tma TBA_TMA_CFG=1"; do
    env $cfg timeout 300 $B --workload $w 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print('$w', '$cfg' or 'default', round(k['fwd_ms'],4), round(k['fwd_gbs']), round(k['bwd_ms'],4))"
  done
done
done
