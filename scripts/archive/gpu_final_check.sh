# Final check at HEAD: every GPU test, smoke, sanitizers (incl. the dH split-K cases), default bench line.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
bash scripts/gpu_sanitize.sh 2>&1 | tail -16
timeout 600 python bench.py > gpurun_out/bench_final_default.json 2> gpurun_out/bench_final_default.err
python -c "
import json; d=json.load(open('gpurun_out/bench_final_default.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['cpu_baseline']['value'], d['clocks'])"
