#!/bin/bash
# Round-2 ncu evidence (run on the GPU box after the commands exited 0
# without ncu): the C3 step's launch list, full captures of its top kernels,
# the 512^3 dilation pass, the general dilation passes and the C4 overlay.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
OUT=gpurun_out/r2
mkdir -p $OUT
# launch list of two C3 steps (warm-up + timed)
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/c3_launches.csv python scripts/profile_pass.py C3 > $OUT/c3_launches.log 2>&1
# full captures of the C3 step's top kernels (second step: -s skips the warm-up's)
ncu --set full --import-source on --clock-control none -k regex:k_seg2_rows -s 3 -c 2 \
    -o $OUT/c3_seg2 python scripts/profile_pass.py C3 > $OUT/c3_seg2.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_bp_cluster -s 4 -c 1 \
    -o $OUT/c3_bp python scripts/profile_pass.py C3 > $OUT/c3_bp.log 2>&1
# the 512^3 fused dilation pass (roofline kernel), one launch
REPS=3 ncu --set full --clock-control none -k regex:k_mark_dilate_plane -s 1 -c 1 \
    -o $OUT/dilate512 python scripts/profile_dilate.py > $OUT/dilate512.log 2>&1
# general dilation passes at 512^3 (x, y, z)
ncu --set full --clock-control none -k regex:k_sdil -s 3 -c 3 \
    -o $OUT/sdil512 python scripts/tl_dilate.py > $OUT/sdil512.log 2>&1
# the C4 overlay tick kernel
ncu --set full --clock-control none -k regex:k_overlay_fused -c 2 \
    -o $OUT/overlay python scripts/sanitize_run.py > $OUT/overlay.log 2>&1
ls -la $OUT
