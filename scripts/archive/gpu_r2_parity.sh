# Round-2 parity: full-size oracle coverage, hostile inputs, one-call schedules vs oracle.
mkdir -p gpurun_out
echo "cores: $(nproc) affinity: $(python -c 'import os; print(len(os.sched_getaffinity(0)))')"; grep -m1 "model name" /proc/cpuinfo; free -g | head -2
TBA_PARITY_OUT=gpurun_out/parity_r02.json timeout 3000 python -m pytest -q -m gpu --durations=30 \
  tests/test_gpu_hostile.py tests/test_gpu_fullsize.py "tests/test_gpu_fused.py::test_one_call_schedules_against_oracle" 2>&1 | tail -60
