# compute-sanitizer over the small C-ABI cases. Output -> gpurun_out/sanitize_<tool>.log
# initcheck runs unfiltered so torch's read-back of every dlogits element is checked too.
# racecheck runs twice: with the single-SM backward GEMMs (TBA_LMB_2SM=0), and with the default
# cta_group::2 GEMMs, whose paired tcgen05.alloc writes the TMEM address into the same shared-memory
# slot of both CTAs (the documented contract) — racecheck reports that as a cross-CTA hazard.
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  if [ $tool = initcheck ]; then F=""; else F="--kernel-name regex=row_|seq_head|tbap_head|tb_fused|tb_finish|lmhead_|lmb_|tc_gemm"; fi
  E=""; if [ $tool = racecheck ]; then E="TBA_LMB_2SM=0"; fi
  env $E timeout 900 compute-sanitizer --tool $tool $F --error-exitcode 9 python scripts/sanitize_case.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool ($E) rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|sanitize cases done" gpurun_out/sanitize_$tool.log | tail -2
done
timeout 900 compute-sanitizer --tool racecheck --kernel-name regex=tc_gemm2 python scripts/sanitize_case.py > gpurun_out/sanitize_racecheck_pair.log 2>&1
echo "racecheck (pair GEMMs) rc=$?"; grep -E "RACECHECK SUMMARY" gpurun_out/sanitize_racecheck_pair.log
grep -oE "in lmhead_bwd.cu:[0-9]+" gpurun_out/sanitize_racecheck_pair.log | sort | uniq -c
# dH split-K (forced on at the small dims, where auto picks S = 1): the slice partials and their reduction
# (initcheck unfiltered, as above: a kernel filter hides the writes of the input generators)
for tool in memcheck initcheck; do
  if [ $tool = initcheck ]; then F=""; else F="--kernel-name regex=lmb_|tc_gemm"; fi
  TBA_LMB_KSPLIT=3 timeout 900 compute-sanitizer --tool $tool $F --error-exitcode 9 python scripts/sanitize_case.py > gpurun_out/sanitize_ksplit_$tool.log 2>&1
  echo "$tool (TBA_LMB_KSPLIT=3) rc=$?"; grep -E "ERROR SUMMARY|sanitize cases done" gpurun_out/sanitize_ksplit_$tool.log | tail -2
done
