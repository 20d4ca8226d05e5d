# compute-sanitizer over the small C-ABI cases. Output -> gpurun_out/sanitize_<tool>.log
# initcheck runs unfiltered so torch's read-back of every dlogits element is checked too.
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  if [ $tool = initcheck ]; then F=""; else F="--kernel-name regex=row_|seq_head|tbap_head|tb_fused|tb_finish|lmhead_|lmb_|tc_gemm"; fi
  timeout 900 compute-sanitizer --tool $tool $F --error-exitcode 9 python scripts/sanitize_case.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|sanitize cases done" gpurun_out/sanitize_$tool.log | tail -2
done
