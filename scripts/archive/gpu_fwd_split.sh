mkdir -p gpurun_out
TBA_LM_MC=5 timeout 600 python -m pytest tests/test_gpu_lmhead.py tests/test_gpu_lmhead_bwd.py -x -q 2>&1 | tail -2
for m in 1 5 1 5; do TBA_LM_MC=$m timeout 600 python bench.py --objective lmhead --steps 6 --warmup 3 --no-e2e --no-cpu-baseline --no-variants 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('MC=$m lmhead fwd', round(d['ms_per_step'],2), round(d['roofline']['achieved']), d['clocks'])"; TBA_LM_MC=$m timeout 300 python scripts/lm_bwd_probe.py --one-call --reps 4; done
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed"
TBA_LM_MC=5 timeout 300 ncu --metrics $M -k regex:lmhead_fwd -c 2 --clock-control none --csv --log-file gpurun_out/fwd_split.csv python scripts/lm_bwd_probe.py --one-call > /dev/null 2>&1
python scripts/ncu_table.py gpurun_out/fwd_split.csv
