"""Short device-resident run for ncu: seeds a bench workload, uploads it, steps a few ticks.

    ncu --profile-from-start off ... python profiles/profile_target.py --workload c2 --ticks 8

Only the last `--ticks` ticks (plain launches, one kernel per phase) lie between cuProfilerStart /
cuProfilerStop; without `--profile-from-start off` ncu also sees the warm-up ticks (graph launches).
"""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_1803_04782_b200 import socfield as sf  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c2")
ap.add_argument("--ticks", type=int, default=8)
ap.add_argument("--warm", type=int, default=30)
args = ap.parse_args()
w = bench.WORKLOADS[args.workload]
engine, P = bench.make_resident(sf, w, 0)
engine.step_resident(args.warm)      # let the crowd start moving (graph launches)
cu = ctypes.CDLL("libcuda.so.1")
cu.cuProfilerStart()
m = engine.step_resident(args.ticks, True)  # plain launches, one kernel per phase
cu.cuProfilerStop()
print("moved per tick:", [x.moved for x in m])
k5 = [x.phase_us[4] for x in m]
print("k5 us per tick: avg %.1f min %.1f" % (sum(k5) / len(k5), min(k5)))
