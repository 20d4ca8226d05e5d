# Correctness of the cluster-multicast LM-head variant, then A/B against the single-CTA one.
TBA_LM_MC=2 timeout 600 python -m pytest tests/test_gpu_lmhead.py -q -x 2>&1 | tail -3
run() {
  env "$@" timeout 300 python bench.py --objective lmhead --steps 10 --warmup 3 --no-e2e --no-cpu-baseline \
    --no-variants 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('%-32s ms=%.2f  TF/s=%.0f  sm_mhz=%s loss=%r' % ('$*', d['ms_per_step'], d['roofline']['achieved'], d['clocks']['sm_mhz'], d['loss']))"
}
for rep in 1 2 3; do
  run TBA_LM_MC=1
  run TBA_LM_MC=2
  run TBA_LM_MC=2 TBA_LM_SWZ=64
done
