# dH split-K on the pair kernel (TBA_LMB_KSPLIT): parity, A/B of the one-call Qwen step, launch list.
TAG=${1:-r01}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_lmhead_bwd.py -x -q 2>&1 | tail -4
for ks in 1 0 1 0; do echo "KSPLIT=$ks"; TBA_LMB_KSPLIT=$ks timeout 300 python scripts/lm_bwd_probe.py --one-call --reps 4; done
for ks in 1 0; do echo "rhomath KSPLIT=$ks"; TBA_LMB_KSPLIT=$ks timeout 300 python scripts/lm_bwd_probe.py --workload rhomath --one-call --reps 4; done
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed"
timeout 400 ncu --metrics $M -k regex:"tc_gemm|lmb_dz|lmb_splitk" -c 6 --clock-control none --csv --log-file gpurun_out/ksplit_${TAG}.csv python scripts/lm_bwd_probe.py --one-call > /dev/null 2>&1
python scripts/ncu_table.py gpurun_out/ksplit_${TAG}.csv
