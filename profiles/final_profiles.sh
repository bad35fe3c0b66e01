#!/bin/bash
# Round-2 evidence set, run on the GPU box: ncu launch list of the bench command, one --set full capture of
# each headline k-5 kernel (summary = per-source-line shares, metrics = the raw page's key counters).
set -u
mkdir -p gpurun_out
[ "${SKIP_LAUNCHES:-0}" = 1 ] || ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file gpurun_out/r2_launches_bench.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-configs > gpurun_out/r2_launches_bench.out 2>&1
DEFAULT_SPECS=("c2 k5_pairs r2_k5_pairs_c2" "c4r k5_pairs r2_k5_pairs_c4r" "paper1000 k5_pairs r2_k5_pairs_paper1000" "c3 k5_field r2_k5_field_c3" "c5 k5_field r2_k5_field_c5")
# FIELD_ONLY=1 re-captures just the large-field kernel (after a change that touched only sfc_k5_writeback.cu)
[ "${FIELD_ONLY:-0}" = 1 ] && DEFAULT_SPECS=("c3 k5_field r2_k5_field_c3" "c5 k5_field r2_k5_field_c5")
for spec in "${DEFAULT_SPECS[@]}"; do
  set -- $spec
  bash profiles/profile_k5.sh $1 $2 $3
  python - "$3" <<'PY'
import csv, io, subprocess, sys
tag = sys.argv[1]
raw = subprocess.run(["ncu", "-i", f"gpurun_out/{tag}.ncu-rep", "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u, v = rows[0], rows[1], rows[2]
keep = ("gpu__time_duration", "launch__", "dram__bytes", "dram__throughput", "lts__t_sectors.sum", "lts__t_bytes", "l1tex__data_bank_conflicts",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared", "smsp__inst_executed.sum", "smsp__inst_executed_pipe", "smsp__issue_active", "sm__warps_active",
        "sm__throughput", "smsp__thread_inst_executed_per_inst", "sm__inst_executed_pipe_fp64", "sm__pipe_fp64", "sm__pipe_alu", "sm__pipe_fma",
        "smsp__average_warps_issue_stalled", "sm__maximum_warps_per_active_cycle_pct", "smsp__warps_eligible")
with open(f"gpurun_out/{tag}.metrics.txt", "w") as f:
    for name, unit, val in zip(h, u, v):
        if name.startswith(keep) or name in ("Kernel Name", "Grid Size", "Block Size"):
            f.write(f"{name} [{unit}] = {val}\n")
PY
done
