# A/B 5 (same box, interleaved): product vs persistent forward row groups vs no token exclusion vs
# the round-1 library (build/r1).
mkdir -p gpurun_out
python scripts/ab_variants.py noexcl=TBA_AB_NO_EXCL persist=TBA_AB_PERSIST_FWD > /dev/null 2>&1
for rep in 1 2 3; do
for v in prod persist noexcl r1; do
  if [ $v = prod ]; then L=""; elif [ $v = r1 ]; then L="$PWD/build/r1/libtba.so"; else L="/tmp/tba_variants/$v/libtba.so"; fi
  for wl in qwen_shard pythia rhomath; do
    TBA_LIBRARY=$L timeout 600 python bench.py --workload $wl --no-e2e --no-cpu-baseline --no-variants > gpurun_out/ab5_${v}_$wl.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/ab5_${v}_$wl.json')); k=d['kernels']
print('$v', '$wl', round(d['ms_per_step'],4), 'fwd', round(k['fwd_ms'],4), 'bwd', round(k['bwd_ms'],4), d['clocks']['sm_mhz'])"
  done
done
done
for wl in pythia redteam pythia_fp32; do
  timeout 600 python bench.py --workload $wl --no-e2e > gpurun_out/bench_r02_$wl.json 2>gpurun_out/bench_r02_$wl.err; tail -c 300 gpurun_out/bench_r02_$wl.json
done
