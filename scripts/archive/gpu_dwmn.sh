mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_lmhead_bwd.py -x -q 2>&1 | tail -4
for m in 1 0 1 0; do TBA_LMB_DW_MN=$m timeout 300 python scripts/lm_bwd_probe.py --one-call --reps 4; done
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed"
timeout 300 ncu --metrics $M -k regex:"tc_gemm|lmb_dz|lmb_gather" -c 6 --clock-control none --csv --log-file gpurun_out/dwmn.csv python scripts/lm_bwd_probe.py --one-call > /dev/null 2>&1
python scripts/ncu_table.py gpurun_out/dwmn.csv
