"""DRAM traffic of the k-5 kernels per workload, from a light ncu pass (one pass, no kernel replay):

    python profiles/traffic.py c2 c1 paper1000 c3 c4r c4 c5      (on the GPU box; writes gpurun_out/r2_traffic.json)

For each workload: runs profiles/profile_target.py under
`ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none`
restricted to the k-5 kernels, skips the first ticks, and averages bytes per k-5 PHASE (all k-5
kernels of a tick).  bench.py reads the committed copy (profiles/r2_traffic.json) for
`roofline.traffic`; the times in that file are ncu's serialised cold-cache times and are NOT used.
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TICKS = {"c2": 12, "c1": 12, "paper1000": 8, "c3": 4, "c4r": 8, "c4": 4, "c5": 2}
WARM = {"c2": 30, "c1": 30, "paper1000": 30, "c3": 6, "c4r": 10, "c4": 6, "c5": 2}


def capture(workload):
    log = os.path.join(ROOT, "gpurun_out", f"r2_traffic_{workload}.csv")
    cmd = ["ncu", "--profile-from-start", "off", "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum",
           "--clock-control", "none",
           "-k", "regex:k5_", "--csv", "--log-file", log, sys.executable, os.path.join(ROOT, "profiles", "profile_target.py"),
           "--workload", workload, "--ticks", str(TICKS[workload]), "--warm", str(WARM[workload])]
    subprocess.run(cmd, check=True, stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
    rows = [r for r in csv.reader(io.StringIO("".join(l for l in open(log) if not l.startswith("=="))))]
    head = rows[0]
    ki, mi, vi, ui = head.index("Kernel Name"), head.index("Metric Name"), head.index("Metric Value"), head.index("Metric Unit")
    idi = head.index("ID")
    launches = {}
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        val = float(r[vi].replace(",", ""))
        unit = r[ui]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "ms": 1e3, "second": 1e6, "s": 1e6}.get(unit, 1)
        launches.setdefault(int(r[idi]), {"kernel": r[ki].split("(")[0]})[r[mi]] = val * scale
    ordered = [launches[k] for k in sorted(launches)]
    kernels = sorted({l["kernel"] for l in ordered})
    tail, n_ticks = ordered, TICKS[workload]  # (only the plain-launch ticks lie inside cuProfilerStart / Stop)
    rd = sum(l.get("dram__bytes_read.sum", 0.0) for l in tail) / n_ticks
    wr = sum(l.get("dram__bytes_write.sum", 0.0) for l in tail) / n_ticks
    us = sum(l.get("gpu__time_duration.sum", 0.0) for l in tail) / n_ticks
    return {"dram_read_bytes_per_k5_phase": rd, "dram_write_bytes_per_k5_phase": wr, "ncu_us_per_k5_phase": us,
            "kernels": kernels, "k5_launches_seen": len(ordered), "ticks_averaged": n_ticks,
            "source": f"profiles/r2_traffic_{workload}.csv"}


def main():
    out_path = os.path.join(ROOT, "gpurun_out", "r2_traffic.json")
    out = json.load(open(out_path)) if os.path.exists(out_path) else {}
    for w in sys.argv[1:]:
        out[w] = capture(w)
        print(w, json.dumps(out[w]), flush=True)
        with open(out_path, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
