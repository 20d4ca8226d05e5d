# A/B of LDG forward configurations. Usage: bash scripts/gpu_ab_ldg.sh [cfgs...]
run() { env "$@" timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print('$*', round(d['ms_per_step'],3), 'fwd', round(k['fwd_ms'],3), round(k['fwd_gbs']), 'bwd', round(k['bwd_ms'],3), round(k['bwd_gbs']), d['clocks']['sm_mhz'], d['clocks']['reasons'])"; }
for c in ${@:-0 1 2 3 4 5 6 7}; do run TBA_FWD_IMPL=ldg TBA_LDG_CFG=$c; done
