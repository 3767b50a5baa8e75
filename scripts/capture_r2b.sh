#!/bin/bash
# Round-2 (late) ncu evidence (run on the GPU box after the commands exited 0
# without ncu): the C3 step's launch list, full captures of its top kernels,
# the 512^3 dilation pass, the general dilation passes and the C4 overlay.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
OUT=gpurun_out/r2b
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
    -o $OUT/overlay python scripts/overlay_tick.py > $OUT/overlay.log 2>&1
ls -la $OUT
# the C5 batch kernels (one 128-target chunk)
ncu --set full --clock-control none -k regex:"k_bq_(tail|seg2)" -s 2 -c 2 \
    -o $OUT/bq python scripts/profile_batch.py 128 > $OUT/bq.log 2>&1
# JSON summaries here (the reports are large; profiles/ keeps the summaries)
for r in c3_seg2 c3_bp dilate512 sdil512 overlay bq; do
  [ -f $OUT/$r.ncu-rep ] && python scripts/ncu_summary.py $OUT/$r.ncu-rep "scripts/capture_r2b.sh ($r)" "round 2, late" > $OUT/$r.json
done
python - <<'PY'
import csv, collections
rows = list(csv.reader(open("gpurun_out/r2b/c3_launches.csv")))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hdr]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
tot = collections.defaultdict(float); cnt = collections.Counter()
for r in rows[hdr + 1:]:
    if len(r) > vi and r[vi]:
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        k = r[ki].split("(")[0].split("<")[0]
        tot[k] += v; cnt[k] += 1
with open("gpurun_out/r2b/c3_launches_summary.txt", "w") as f:
    s = sum(tot.values())
    f.write(f"C3 launch list (2 steps, ncu gpu__time_duration, serialised, cold): total {s/1e3:.1f} us\n")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        f.write(f"{v/1e3:10.1f} us {100*v/s:5.1f}% {cnt[k]:5d} launches  {k}\n")
PY
rm -f $OUT/sdil512.ncu-rep $OUT/overlay.ncu-rep $OUT/dilate512.ncu-rep $OUT/bq.ncu-rep
ls -la $OUT
