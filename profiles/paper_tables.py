"""The paper's running-time tables on the B200 engine, through the reference's own
sweep harness (socfield.run_bench = reference bench.cpp:65-111 on the CUDA engine).

Baseline scenario of all three: 1000 x 1000 su, density 0.5, eight directions, 1000 ticks in the paper;
here `--ticks` ticks per run (default 20), scaled to the paper's 1000 in the "s / 1000 ticks" column.

    multi-step sum   fields 7x7 ... 77x77 (ratios 1, 3, ..., 11)          paper: 62 ... 3238 s
    walk period      maximal period 1, 3, ..., 11                          paper: 62 ... 64 s
    combo            pedestrian geometry 1x1 ... 11x11 x walk period       paper: 63.5 ... 264.6 s

    python profiles/paper_tables.py --out profiles/r2_paper_tables.csv [--ticks 20] [--tables sum,period,combo]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1803_04782_b200 import socfield as sf  # noqa: E402

PAPER = {
    "sum": {1: 62, 3: 317, 5: 738, 7: 1424, 9: 2187, 11: 3238},
    "period": {1: 62, 3: 64, 5: 64, 7: 63, 9: 62, 11: 62},
    "combo": {(1, 1): 63.5, (3, 1): 264.6, (5, 1): 213.5, (7, 1): 207.7, (9, 1): 197.6, (11, 1): 201.5,
              (1, 11): 63.9, (3, 11): 261.8, (5, 11): 200.8, (7, 11): 193.8, (9, 11): 182.1, (11, 11): 189.6},
}

ap = argparse.ArgumentParser()
ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "paper_tables.csv"))
ap.add_argument("--ticks", type=int, default=20)
ap.add_argument("--tables", default="sum,period,combo")
ap.add_argument("--grid", type=int, default=1000)
args = ap.parse_args()
base = sf.parse_scenario(f"grid = {args.grid}x{args.grid}\ndensity = 0.5\ndirections = eight\nfield_geometry = 7x7\n"
                         "seed = 42\nrebuild_interval = 50\n")
lines = ["table,key,population,field_geometry,pedestrian_geometry,walk_period_max,sf,ticks,device_ms_per_tick,"
         "device_s_per_1000_ticks,host_run_ms_per_tick,ped_steps_per_s,paper_s_per_1000_ticks,speedup_vs_paper,status"]


def emit(table, key, r, paper):
    tick_ms = r["device_mean_ms"] / max(r["ticks"], 1)
    s1000 = tick_ms  # ms per tick == s per 1000 ticks
    lines.append(",".join(str(x) for x in (
        table, key, r["population"], "%dx%d" % r["field_geometry"], "%dx%d" % r["pedestrian_geometry"], r["walk_period_max"],
        r["sf"], r["ticks"], "%.4f" % tick_ms, "%.3f" % s1000, "%.4f" % (r["mean_ms"] / max(r["ticks"], 1)),
        "%.4g" % r["ped_steps_per_s"], paper if paper is not None else "", ("%.1f" % (paper / s1000)) if paper and s1000 > 0 else "",
        r["status"].replace(",", ";"))))
    print(lines[-1], flush=True)


t0 = time.time()
if "sum" in args.tables:
    rows, _ = sf.run_bench(base, field_ratios=[1, 3, 5, 7, 9, 11], ticks=args.ticks, repeats=1, warmup=True)
    for ratio, r in zip([1, 3, 5, 7, 9, 11], rows):
        emit("multi-step-sum", ratio, r, PAPER["sum"][ratio])
if "period" in args.tables:
    rows, _ = sf.run_bench(base, walk_period_maxes=[1, 3, 5, 7, 9, 11], ticks=args.ticks, repeats=1, warmup=True)
    for period, r in zip([1, 3, 5, 7, 9, 11], rows):
        emit("walk-period", period, r, PAPER["period"][period])
if "combo" in args.tables:
    geoms = [(1, 1), (3, 3), (5, 5), (7, 7), (9, 9), (11, 11)]
    periods = [1, 11]
    rows, _ = sf.run_bench(base, walk_period_maxes=periods, pedestrian_geometries=geoms, ticks=args.ticks, repeats=1, warmup=True)
    i = 0
    for period in periods:  # (pedestrian geometry is the innermost axis of the sweep)
        for g in geoms:
            emit("combo", f"{g[0]}x{g[1]}/T{period}", rows[i], PAPER["combo"].get((g[0], period)))
            i += 1
os.makedirs(os.path.dirname(args.out), exist_ok=True)
with open(args.out, "w") as f:
    f.write("\n".join(lines) + "\n")
print(f"wrote {args.out} in {time.time() - t0:.0f} s")
