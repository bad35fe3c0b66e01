"""Scenario texts and hand-built populations shared by the parity tests.

The texts use the reference's `key = value` scenario format (reference
proj/src/scenario.cpp:172-268); the fixtures restate those of the reference's own tests
(proj/tests/unit/test_engine.cpp, proj/tests/acceptance/acceptance_main.cpp).
"""
import itertools

DESK64 = """# desk-scale validation scenario (reference proj/scenarios/desk64.scn)
grid = 64x64
density = 0.5
directions = eight
field_geometry = 7x7
pedestrian_geometry = 1x1
walk_period = 1..3
ticks = 100
seed = 42
"""

SEQPAR24 = """# reference test_engine.cpp:352-360
grid = 24x24
density = 0.4
directions = four
walk_period = 1..3
seed = 99
rebuild_interval = 10
"""


def acceptance3_scenarios():
    """The 24 scenarios of acceptance criterion 3 (acceptance_main.cpp:60-89)."""
    out = []
    seed = 1000
    for density, dirs, ped in itertools.product((0.1, 0.5, 0.9), ("uni", "bi", "four", "eight"), (1, 3)):
        out.append((f"d{density}-{dirs}-ped{ped}",
                    f"grid = 64x64\ndensity = {density}\ndirections = {dirs}\npedestrian_geometry = {ped}x{ped}\n"
                    f"walk_period = 1..3\nseed = {seed}\nrebuild_interval = 50\n"))
        seed += 1
    return out


def variant(text: str, **overrides) -> str:
    """Scenario text with keys replaced / appended."""
    lines = [l for l in text.splitlines() if l.split("=")[0].strip() not in overrides]
    lines += [f"{k} = {v}" for k, v in overrides.items()]
    return "\n".join(lines) + "\n"


EXTRA = {
    "closed-four": "grid = 32x20\nboundary = closed\ndensity = 0.4\ndirections = four\nseed = 13\nrebuild_interval = 7\n",
    "closed-ped3": "grid = 40x40\nboundary = closed\ndensity = 0.3\ndirections = eight\npedestrian_geometry = 3x3\n"
                   "walk_period = 1..2\nseed = 5\nrebuild_interval = 0\n",
    "field21": "grid = 48x40\ndensity = 0.2\ndirections = eight\nfield_geometry = 21x21\nwalk_period = 1..3\nseed = 77\n"
               "rebuild_interval = 9\n",
    "field-5x9": "grid = 37x29\ndensity = 0.3\ndirections = bi\nfield_geometry = 5x9\nseed = 3\nrebuild_interval = 4\n",
    "field-bigger-than-grid": "grid = 8x6\ndensity = 0.2\ndirections = eight\nfield_geometry = 11x9\nseed = 8\n"
                              "rebuild_interval = 3\n",
    "linear-regulation": "grid = 40x40\ndensity = 0.5\ndirections = eight\nregulation = linear\ndensity_radius = 2\n"
                         "walk_period = 1..3\nseed = 21\nrebuild_interval = 0\n",
    "linear-closed": "grid = 30x30\nboundary = closed\ndensity = 0.6\ndirections = four\nregulation = linear\n"
                     "density_radius = 3\nseed = 22\nrebuild_interval = 5\n",
    "k2": "grid = 32x32\ndensity = 0.5\nchunk_k = 2\nseed = 31\nrebuild_interval = 0\n",
    "k4": "grid = 32x32\ndensity = 0.5\nchunk_k = 4\nseed = 31\nrebuild_interval = 0\n",
    "k16": "grid = 32x32\ndensity = 0.5\nchunk_k = 16\nseed = 31\nrebuild_interval = 0\n",
    "weights": "grid = 33x31\ndensity = 0.45\ndirections = eight\nweight_static = 0.5\nweight_dir_attractive = 0.25\n"
               "weight_dir_repulsive = 1.75\nweight_recurrent = 0.6\ngoal_bias = 0.35\nfield_gain = 1.3\n"
               "field_decay = -0.37\nwalk_period = 1..4\nseed = 17\nrebuild_interval = 6\n",
    "ped5": "grid = 64x48\ndensity = 0.35\ndirections = eight\npedestrian_geometry = 5x3\nfield_geometry = 9x9\n"
            "walk_period = 1..2\nseed = 4\nrebuild_interval = 8\n",
    # sparse crowds on ragged grids: most k-5 tiles see no mover in a tick (active-tile list, wrap-around marking)
    "sparse-periodic": "grid = 203x117\ndensity = 0.004\ndirections = eight\nwalk_period = 1..2\nseed = 61\nrebuild_interval = 12\n",
    "sparse-closed": "grid = 150x90\nboundary = closed\ndensity = 0.006\ndirections = four\nseed = 62\nrebuild_interval = 9\n",
    "sparse-field15": "grid = 160x96\ndensity = 0.003\ndirections = eight\nfield_geometry = 15x11\nseed = 63\nrebuild_interval = 0\n",
    # large fields: the region of a 32 x 16 k-5 tile exceeds one staging pass (chunked staging, one event list) ...
    "field35": "grid = 97x83\ndensity = 0.03\ndirections = eight\nfield_geometry = 35x35\nwalk_period = 1..2\nseed = 71\n"
               "rebuild_interval = 4\n",
    # ... and, in a crowd, the events of a region overflow the list (per-walk re-staging)
    "field41-crowd": "grid = 90x75\ndensity = 0.7\ndirections = eight\nfield_geometry = 41x41\nseed = 72\nrebuild_interval = 0\n",
    # 13 x 13 fields (168 offsets): beyond the list-walk-alone range, within the list walk's range as the dense kernel
    "field13-crowd": "grid = 70x45\ndensity = 0.5\ndirections = eight\nfield_geometry = 13x13\nwalk_period = 1..2\nseed = 81\n"
                     "rebuild_interval = 6\n",
    "wide-ragged": "grid = 131x67\ndensity = 0.3\ndirections = bi\nwalk_period = 1..3\nseed = 123\nrebuild_interval = 10\n",
}


# ---- BASELINE.json configs at (or shaped like) their stated parameters ------------------------
# c1 and c2 are the configs themselves over their full / a long horizon; c3, c4 and c5 keep the
# config's density, field geometry, regulation and obstacle share on a grid the CPU reference can
# hold and finish (SURVEY.md 8c "scale limits").  Reference-recorded digests of each live in
# tests/golden/baseline_shaped.json (tests/golden/make_golden.py --big).
C1_TEXT = ("grid = 200x200\nboundary = closed\ndensity = 0.0125\ndirections = uni\nfield_geometry = 7x7\n"
           "seed = 42\nrebuild_interval = 50\n")
C1_EXIT = [(0, 399, 399, 1.0, -0.02, 199, 100)]  # one omni-attractive field anchored at the exit su, reaching the whole room
C2_TEXT = ("grid = 2000x500\nboundary = periodic\ndensity = 0.02\ndirections = bi\nwalk_period = 1..3\n"
           "field_geometry = 7x7\nseed = 42\nrebuild_interval = 50\n")


def obstacle_anchors(width, height, share=0.01, seed=7):
    """7 x 7 omni-repulsive static fields on `share` of the su; positions from a seeded 64-bit LCG
    (self-contained: no dependence on a numpy bit-generator's stream)."""
    n = int(round(share * width * height))
    seen, out, x = set(), [], seed
    while len(out) < n:
        x = (x * 6364136223846793005 + 1442695040888963407) % (1 << 64)
        at = (x >> 33) % (width * height)
        if at in seen:
            continue
        seen.add(at)
        out.append((1, 7, 7, 1.0, -0.5, at % width, at // width))
    return out


BASELINE_SHAPED = {
    "c1-full": dict(text=C1_TEXT, static=C1_EXIT, ticks=[100, 500, 1000]),
    "c2-100": dict(text=C2_TEXT, static=[], ticks=[1, 10, 50, 100]),
    # c3: 35 x 35 fields (1224 support offsets) at rho 200000 / 2^26, two rebuilds inside the horizon
    "c3-1024": dict(text="grid = 1024x1024\ndensity = 0.00298023223876953125\ndirections = eight\nfield_geometry = 35x35\n"
                         "seed = 42\nrebuild_interval = 2\n", static=[], ticks=[2, 4]),
    # c4: 7 x 7 fields at rho 10^6 / 2^30 (one mover per ~1000 su: active-tile list), two rebuilds
    "c4-4096": dict(text="grid = 4096x4096\ndensity = 0.000931322574615478515625\ndirections = eight\nfield_geometry = 7x7\n"
                         "seed = 42\nrebuild_interval = 6\n", static=[], ticks=[6, 12]),
    # c5: 77 x 77 fields (5928 offsets) WITH linear regulation r = 3 and 7 x 7 obstacle fields on 1 % of the su, rho 0.05
    "c5-256": dict(text="grid = 256x192\ndensity = 0.05\ndirections = eight\nfield_geometry = 77x77\nregulation = linear\n"
                        "density_radius = 3\nseed = 42\nrebuild_interval = 4\n", static=obstacle_anchors(256, 192), ticks=[3, 6]),
}
