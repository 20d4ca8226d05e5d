# cta_group::2 LM-head variant: debug check, parity tests, then A/B against the single-SM kernel.
TBA_LM_MC=3 timeout 120 python scripts/lmhead_debug.py 2>&1 | tail -6
TBA_LM_MC=3 timeout 600 python -m pytest tests/test_gpu_lmhead.py -q -x 2>&1 | tail -3
run() {
  env "$@" timeout 300 python bench.py --objective lmhead --steps 10 --warmup 3 --no-e2e --no-cpu-baseline \
    --no-variants 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('%-32s ms=%.2f  TF/s=%.0f  sm_mhz=%s loss=%r' % ('$*', d['ms_per_step'], d['roofline']['achieved'], d['clocks']['sm_mhz'], d['loss']))"
}
for rep in 1 2 3; do
  run TBA_LM_MC=1
  run TBA_LM_MC=3
  run TBA_LM_MC=3 TBA_LM_SWZ=16
done
