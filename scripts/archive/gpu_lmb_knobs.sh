# A/B of the LM-head backward raster / policy / chunk knobs (CUDA events, back to back).
P="timeout 300 python scripts/lm_bwd_probe.py --reps 5"
$P
TBA_LMB_NINNER=0 $P
TBA_LMB_NINNER=1 $P
TBA_LMB_NINNER=2 $P
TBA_LMB_NINNER=0 TBA_LMB_SWZ=16 $P
TBA_LMB_POL=2 $P
TBA_LMB_POL=8 $P
$P --chunk 8192
TBA_LMB_POL=8 $P --chunk 8192
$P --chunk 32768
$P --chunk 65536
$P
