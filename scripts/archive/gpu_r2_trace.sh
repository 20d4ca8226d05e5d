# Phase trace of the deferred row pass at the Qwen shard (TBA_AB_DEFER_TRACE build)
mkdir -p gpurun_out
python scripts/ab_variants.py trace=TBA_AB_DEFER_TRACE > /dev/null 2>&1
TBA_LIBRARY=/tmp/tba_variants/trace/libtba.so timeout 600 python scripts/defer_trace.py
