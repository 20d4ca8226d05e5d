# Round-2 evidence at HEAD: every GPU test (parity maxima -> gpurun_out/parity_r02.json), the
# confident-sequence test against the no-exclusion A/B build (expected to fail), smoke, bench lines
# (default, small shapes, deferred, TBA', strong N=1, the N>1 flows on one GPU), the reference arm,
# ncu launch list + DRAM bytes + --set full captures, compute-sanitizer on the default path.
mkdir -p gpurun_out
python scripts/ab_variants.py noexcl=TBA_AB_NO_EXCL > /dev/null 2>&1
TBA_PARITY_OUT=gpurun_out/parity_r02.json timeout 2400 python -m pytest tests -q -m gpu 2>&1 | tail -4
echo "== confident sequences with the no-exclusion build (expected: fail)"
TBA_LIBRARY=/tmp/tba_variants/noexcl/libtba.so timeout 600 python -m pytest -q tests/test_gpu_hostile.py -k confident 2>&1 | grep -E "AssertionError|passed|failed" | head -4
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_r02_qwen_shard.json 2> gpurun_out/bench_r02_qwen_shard.err; tail -c 600 gpurun_out/bench_r02_qwen_shard.json
for wl in pythia redteam rhomath toy gsm8k_t3 gsm8k_k40 tldr_t4 math_t5_shard pythia_fp32; do
  timeout 600 python bench.py --workload $wl --no-e2e > gpurun_out/bench_r02_$wl.json 2>/dev/null
done
timeout 600 python bench.py --workload qwen_shard --objective tbap --no-e2e --no-cpu-baseline > gpurun_out/bench_r02_qwen_shard_tbap.json 2>/dev/null
for wl in qwen_shard pythia redteam rhomath math_t5_shard gsm8k_t3 pythia_fp32; do
  timeout 600 python bench.py --workload $wl --schedule deferred --no-e2e --no-cpu-baseline > gpurun_out/bench_r02_${wl}_deferred.json 2>/dev/null
done
timeout 600 python bench.py --workload toy --cuda-graph --no-e2e --no-cpu-baseline > gpurun_out/bench_r02_toy_graph.json 2>/dev/null
timeout 900 python bench.py --scaling strong --workload qwen --steps 5 --warmup 3 > gpurun_out/bench_r02_qwen_strong.json 2>/dev/null
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 2 --steps 5 --warmup 3 --workload qwen_shard --dist-backend gloo --share-gpu --no-variants --no-e2e > gpurun_out/bench_r02_n2_gloo_shared.json 2>/dev/null
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 \
  bench.py --gpus 2 --steps 3 --warmup 3 --workload rhomath --scaling strong --chunk-groups 4 --dist-backend gloo --share-gpu > gpurun_out/bench_r02_n2_strong_rhomath_gloo_shared.json 2>/dev/null
timeout 900 python bench.py --impl reference > gpurun_out/bench_r02_reference.json 2>/dev/null
python - <<'PY'
import json, glob
for f in sorted(glob.glob('gpurun_out/bench_r02_*.json')):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, 'ERR', e); continue
    r = d.get('roofline') or {}
    print(f.split('bench_r02_')[1][:-5], round(d['value']), round(d['ms_per_step'], 4), 'frac', r.get('frac') and round(r['frac'], 3),
          (d.get('kernels') or {}).get('fwd_frac') and round(d['kernels']['fwd_frac'], 3), (d.get('kernels') or {}).get('step_frac') and round(d['kernels']['step_frac'], 3),
          'defer', (d.get('variants') or {}).get('deferred_scale', {}).get('ms_per_step'), (d.get('clocks') or {}).get('sm_mhz'))
PY
bash scripts/gpu_profile.sh r02 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:row_single -s 3 -c 1 -o gpurun_out/prof_row_single1_r02 -f python bench.py --no-e2e --no-cpu-baseline --no-variants --workload qwen_group --schedule deferred --steps 1 --warmup 3 > /dev/null 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:row_single -s 3 -c 2 --csv --log-file gpurun_out/dram_deferred_r02.csv python bench.py --no-e2e --no-cpu-baseline --no-variants --schedule deferred --steps 2 --warmup 3 > /dev/null 2>&1
# compute-sanitizer is closed on the GPU pool (round 2): tests/test_gpu_guard.py is the bounds check
ls gpurun_out | head -80
