#!/bin/bash
# ncu --set full of the two rebuild passes (check, commit) of one workload: profiles/profile_rebuild.sh <workload>
w=${1:-c4r}
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:rebuild_kernel -c 2 -o gpurun_out/r2_rebuild_$w -f \
    python profiles/profile_target.py --workload $w --ticks 8 --warm 45 2>&1 | tail -2
ncu -i gpurun_out/r2_rebuild_$w.ncu-rep --page raw --csv > gpurun_out/r2_rebuild_$w.raw.csv 2>/dev/null
python - "$w" <<'PY'
import csv, sys
w = sys.argv[1]
rows = list(csv.reader(open(f"gpurun_out/r2_rebuild_{w}.raw.csv")))
h = rows[0]
keep = ("gpu__time_duration.sum", "launch__grid_size", "launch__registers_per_thread", "launch__occupancy_limit", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__inst_executed.sum", "smsp__issue_active.avg.pct", "sm__warps_active.avg.pct", "smsp__average_warps_issue_stalled", "launch__waves", "sm__maximum_warps_per_active_cycle_pct", "launch__shared_mem_per_block", "launch__occupancy")
with open(f"gpurun_out/r2_rebuild_{w}.metrics.txt", "w") as f:
    for r in rows[2:]:
        f.write("---- launch\n")
        for name, unit, val in zip(h, rows[1], r):
            if name.startswith(keep):
                f.write(f"{name} [{unit}] = {val}\n")
print(open(f"gpurun_out/r2_rebuild_{w}.metrics.txt").read())
PY
python profiles/ncu_lines.py gpurun_out/r2_rebuild_$w.ncu-rep 30 > gpurun_out/r2_rebuild_$w.summary.txt 2>&1
head -45 gpurun_out/r2_rebuild_$w.summary.txt
