"""Per-source-line instruction / stall-sample shares of one kernel in an .ncu-rep (needs -lineinfo).

    python profiles/ncu_lines.py gpurun_out/x.ncu-rep [top_n]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, v = rows[0], rows[2]
for k in ["gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
          "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
          "launch__registers_per_thread", "dram__bytes_read.sum", "dram__bytes_write.sum",
          "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_sectors.sum",
          "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
          "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
          "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
          "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
          "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio",
          "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
          "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
          "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio"]:
    if k in h:
        print(f"{k} = {v[h.index(k)]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur, hdr, agg = None, None, {}
for r in csv.reader(io.StringIO(src)):
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if len(r) > 5 and r[0] == "Line No":
        hdr = r
        ci, ti, sm = hdr.index("Instructions Executed"), hdr.index("Thread Instructions Executed"), hdr.index("# Samples")
        continue
    if hdr and len(r) == len(hdr) and r[0].isdigit() and r[2] == "-":
        try:
            n, t, s = int(r[ci]), int(r[ti]), int(r[sm])
        except ValueError:
            continue
        a = agg.setdefault((cur, int(r[0]), r[1][:96]), [0, 0, 0])
        a[0] += n
        a[1] += t
        a[2] += s
tot = sum(a[0] for a in agg.values()) or 1
ts = sum(a[2] for a in agg.values()) or 1
print("total warp instructions", tot, "samples", ts)
for k, a in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{a[0]:>9} {100 * a[0] / tot:5.1f}% thr {a[1] / max(a[0], 1):5.1f} samp {100 * a[2] / ts:5.1f}% {k[0][:18]}:{k[1]}: {k[2]}")

if len(sys.argv) > 3:  # optional "lo-hi,lo-hi,..." line buckets of the first file
    buckets = [tuple(map(int, b.split("-"))) for b in sys.argv[3].split(",")]
    main_file = max(set(k[0] for k in agg), key=lambda f: sum(a[0] for k, a in agg.items() if k[0] == f))
    for lo, hi in buckets:
        n = sum(a[0] for k, a in agg.items() if k[0] == main_file and lo <= k[1] <= hi)
        smp = sum(a[2] for k, a in agg.items() if k[0] == main_file and lo <= k[1] <= hi)
        print(f"lines {lo}-{hi}: {n} instr ({100 * n / tot:.1f}%), samples {100 * smp / ts:.1f}%")
