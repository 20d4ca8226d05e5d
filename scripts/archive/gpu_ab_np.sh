TBA_FWD_NP=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
run() { w=$1; shift; env $E timeout 600 python bench.py --workload $w --steps 30 --warmup 5 --no-e2e --no-cpu-baseline "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print('$E $w', round(d['ms_per_step'],4), 'fwd', round(k['fwd_ms'],4), round(k['fwd_gbs']))"; }
for i in 1 2; do for n in 0 1 2; do E="TBA_FWD_NP=$n"; run qwen_shard; done; done
for n in 0 1; do E="TBA_FWD_NP=$n"; run rhomath; run pythia; done
