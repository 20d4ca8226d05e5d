mkdir -p gpurun_out
for c in 2 4; do
TBA_SINGLE_CFG=$c ncu --set full --clock-control none --import-source on -k regex:row_single -s 2 -c 1 -o gpurun_out/prof_single_c$c -f python bench.py --schedule deferred --workload qwen_group --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/prof_single_c$c.log 2>&1
tail -1 gpurun_out/prof_single_c$c.log
done
