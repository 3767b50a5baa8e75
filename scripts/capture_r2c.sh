#!/bin/bash
# Round-2 (final) ncu evidence, run on the GPU box after the same commands
# exited 0 without ncu: the C3 step's launch list, a full capture of its top
# kernel (k_seg2_rows, the step's first solve) and the rewritten general
# dilation passes (k_sdil_x / k_sdil_y<32,4> / k_sdil_z<32,4>) on the 512^3
# C5 grid (tl_dilate.py runs 3 C3 dilations of 3 passes first: -s 9).
set -u
cd "$(dirname "$0")/.."
OUT=gpurun_out/r2c
mkdir -p $OUT
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/c3_launches.csv python scripts/profile_pass.py C3 > $OUT/c3_launches.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_seg2_rows -s 3 -c 1 \
    -o $OUT/c3_seg2 python scripts/profile_pass.py C3 > $OUT/c3_seg2.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_sdil -s 9 -c 3 \
    -o $OUT/sdil512 python scripts/tl_dilate.py > $OUT/sdil512.log 2>&1
ls -la $OUT
for r in c3_seg2 sdil512; do
  [ -f $OUT/$r.ncu-rep ] && python scripts/ncu_summary.py $OUT/$r.ncu-rep "scripts/capture_r2c.sh ($r)" "round 2, final" > $OUT/$r.json
done
python - <<'PY'
import csv, collections, re
rows = list(csv.reader(open("gpurun_out/r2c/c3_launches.csv")))
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
        k = r[ki].replace("<unnamed>::", "").replace("(anonymous namespace)::", "")
        k = re.sub(r"^void ", "", k).split("(")[0]
        k = re.sub(r"<.*", "", k)
        tot[k] += v; cnt[k] += 1
with open("gpurun_out/r2c/c3_launches_summary.txt", "w") as f:
    s = sum(tot.values())
    f.write(f"C3 launch list (2 steps: warm-up + timed; ncu gpu__time_duration, serialised, cold caches): total {s/1e3:.1f} us\n")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        f.write(f"{v/1e3:10.1f} us {100*v/s:5.1f}% {cnt[k]:5d} launches  {k}\n")
PY
rm -f $OUT/sdil512.ncu-rep
ls -la $OUT
