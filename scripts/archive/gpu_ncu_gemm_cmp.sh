# ncu --set full: our backward GEMM (dH, chunk 0) and the dz pass vs cuBLAS's dH GEMM on the same shape
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"tc_gemm|lmb_dz_from_z" -c 3 -o gpurun_out/ncu_lmb_full -f python scripts/lm_bwd_probe.py --one-call > gpurun_out/ncu_lmb_full.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:nvjet -s 1 -c 1 -o gpurun_out/ncu_cublas_dh -f python scripts/lm_bwd_probe.py --cublas > gpurun_out/ncu_cublas_dh.log 2>&1
for f in ncu_lmb_full ncu_cublas_dh; do ncu -i gpurun_out/$f.ncu-rep --page raw --csv > gpurun_out/$f.raw.csv 2>/dev/null; ncu -i gpurun_out/$f.ncu-rep --page details --csv > gpurun_out/$f.details.csv 2>/dev/null; done
ls -la gpurun_out | grep ncu
