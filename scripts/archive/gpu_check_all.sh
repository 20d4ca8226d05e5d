timeout 1500 python -m pytest tests -q -m gpu 2>&1 | grep -E "^FAILED|passed|failed" | tail -8
run() { w=$1; shift; timeout 600 python bench.py --workload $w --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-variants "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print('$w $*', round(d['ms_per_step'],4), 'tok/s %.4g' % d['value'], 'fwd', round(k.get('fwd_ms',0),4), round(k.get('fwd_gbs',0)), 'launches', d['gpu_launches'])"; }
for w in toy pythia redteam rhomath qwen_shard; do run $w; done
