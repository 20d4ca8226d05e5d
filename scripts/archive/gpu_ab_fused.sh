run() { w=$1; shift; timeout 600 python bench.py --workload $w --steps 30 --warmup 5 --no-e2e --no-cpu-baseline "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$w $*', round(d['ms_per_step'],4), 'tok/s %.4g' % d['value'], 'step GB/s(6V) %.0f' % d['hbm_gbs_step'], 'roof %.0f %.3f' % (r['achieved'], r['frac']))"; }
for w in toy pythia redteam rhomath qwen_shard; do run $w; run $w --schedule fused; done
for D in 1 2 3 4; do TBA_FUSED_D=$D run pythia --schedule fused; TBA_FUSED_D=$D run redteam --schedule fused; done
