run() { w=$1; shift; env "$@" timeout 600 python bench.py --workload $w --steps 30 --warmup 5 --no-e2e --no-cpu-baseline "${EXTRA[@]}" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print('$w $*', round(d['ms_per_step'],4), 'fwd', round(k['fwd_ms'],4), round(k['fwd_gbs']), 'bwd', round(k['bwd_ms'],4), round(k['bwd_gbs']))"; }
for w in qwen_shard rhomath pythia; do for t in 0 64 128; do run $w TBA_BWD_TPR=$t; done; done
EXTRA=(--objective tbap); run qwen_shard TBA_BWD_TPR=0
