# A/B of the LM-head kernel's work-item size (TBA_LM_G) and L2 raster (TBA_LM_SWZ), interleaved.
run() {
  env "$@" timeout 300 python bench.py --objective lmhead --steps 10 --warmup 3 --no-e2e --no-cpu-baseline \
    --no-variants 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('%-32s ms=%.2f  TF/s=%.0f  sm_mhz=%s' % ('$*', d['ms_per_step'], d['roofline']['achieved'], d['clocks']['sm_mhz']))"
}
for rep in 1 2; do
  run TBA_LM_G=4 TBA_LM_SWZ=16
  run TBA_LM_G=4 TBA_LM_SWZ=8
  run TBA_LM_G=4 TBA_LM_SWZ=32
  run TBA_LM_G=4 TBA_LM_SWZ=64
  run TBA_LM_G=8 TBA_LM_SWZ=16
  run TBA_LM_G=8 TBA_LM_SWZ=32
  run TBA_LM_G=16 TBA_LM_SWZ=32
done
