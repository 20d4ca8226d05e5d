mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_lmhead_bwd.py -x -q 2>&1 | tail -2
for r in 1 2; do timeout 300 python scripts/lm_bwd_probe.py --one-call --reps 4; done
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed"
timeout 300 ncu --metrics $M -k regex:lmhead_fwd -c 2 --clock-control none --csv --log-file gpurun_out/fwd_zstore.csv python scripts/lm_bwd_probe.py --one-call > /dev/null 2>&1
python scripts/ncu_table.py gpurun_out/fwd_zstore.csv
timeout 300 compute-sanitizer --tool memcheck --kernel-name regex=lmhead_fwd python scripts/sanitize_case.py 2>&1 | grep -E "ERROR SUMMARY|done"
