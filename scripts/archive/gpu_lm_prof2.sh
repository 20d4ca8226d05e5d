# LM head: paired fused-vs-cuBLAS bench line, and ncu --set full of the cta_group::2 variant for comparison.
timeout 600 python bench.py --objective lmhead --steps 12 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_lm_paired.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/bench_lm_paired.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['variants'])"
B="python bench.py --objective lmhead --no-e2e --no-cpu-baseline --no-variants"
TBA_LM_MC=3 timeout 900 ncu --set full --clock-control none -k regex:lmhead_fwd -s 3 -c 1 -o gpurun_out/prof_lmhead_fwd_2sm_dbg -f $B --steps 1 --warmup 3 > /dev/null 2>&1
ls -la gpurun_out/prof_lmhead_fwd_2sm_dbg.ncu-rep
