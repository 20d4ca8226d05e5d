# Bench every BASELINE workload (the headline line is qwen_shard, with e2e and cpu_baseline).
mkdir -p gpurun_out
TAG=${1:-r01}
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_${TAG}_qwen_shard.json 2> gpurun_out/bench_${TAG}_qwen_shard.err
for w in toy pythia rhomath redteam; do
  timeout 600 python bench.py --workload $w --steps 50 --warmup 10 --no-e2e --no-cpu-baseline > gpurun_out/bench_${TAG}_$w.json 2> gpurun_out/bench_${TAG}_$w.err
done
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_${TAG}_reference.json 2> gpurun_out/bench_${TAG}_reference.err
for f in gpurun_out/bench_${TAG}_*.json; do echo "$f"; python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1])
k=d.get('kernels',{}); r=d.get('roofline') or {}
print(' value %.4g %s  ms %.4g  fwd %s  bwd %s  frac %s e2e %s cpu %s' % (d['value'], d['unit'], d['ms_per_step'], k.get('fwd_gbs'), k.get('bwd_gbs'), r.get('frac'), (d.get('e2e') or {}).get('value'), (d.get('cpu_baseline') or {}).get('value')))
"; done
