"""Regenerates tests/golden/digests.json from the UNMODIFIED reference.

Run in the build container only (needs /root/reference -> `make -C oracle ref`):

    python tests/golden/make_golden.py

Each entry records the scenario text, the seeded population and the FNV-1a state digest
(occupancy, three dynamic images, centres — reference tests/acceptance/acceptance_main.cpp:39-58)
after the listed tick counts of Engine::run in sequential mode.  The first two entries repeat the
vectors quoted in SURVEY.md §8(c); the rest extend them to the acceptance-3 scenario family and
to the edge cases in tests/scenarios.py.
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import shim  # noqa: E402
from tests import scenarios as sc  # noqa: E402


def record(lib, text, ticks):
    sim = shim.Sim.from_scenario(lib, text, workers=1)
    out = {"scenario": text, "population": sim.population, "digests": []}
    last = 0
    for t in ticks:
        sim.run(t - last)
        last = t
        out["digests"].append([t, f"{sim.digest():#018x}"])
    return out


def record_big(lib, spec):
    """BASELINE-shaped cases: Engine::run in parallel mode on every core (the reference guarantees,
    and its acceptance criterion 3 checks, that the result does not depend on the worker count)."""
    sim = shim.Sim.from_scenario(lib, spec["text"], workers=os.cpu_count() or 1)
    if spec["static"]:
        sim.set_static_fields(spec["static"])
    out = {"scenario": spec["text"], "static_fields": [list(a) for a in spec["static"]], "population": sim.population,
           "digests": [[0, f"{sim.digest():#018x}"]]}
    last = 0
    for t in spec["ticks"]:
        sim.run(t - last, mode="par")
        last = t
        out["digests"].append([t, f"{sim.digest():#018x}"])
        print(f"  tick {t}: {out['digests'][-1][1]}", flush=True)
    return out


def main_big():
    lib = shim.load_ref()
    path = os.path.join(HERE, "baseline_shaped.json")
    golden = json.load(open(path)) if os.path.exists(path) else {}
    only = [a for a in sys.argv[1:] if not a.startswith("--")]
    for name, spec in sc.BASELINE_SHAPED.items():
        if only and name not in only:
            continue
        print(name, flush=True)
        golden[name] = record_big(lib, spec)
        with open(path, "w") as f:
            json.dump(golden, f, indent=1)
    print(f"wrote {len(golden)} entries")


def main():
    if "--big" in sys.argv:
        return main_big()
    lib = shim.load_ref()
    golden = {
        "desk64": record(lib, sc.DESK64, [0, 1, 10, 49, 50, 100]),
        "seqpar24": record(lib, sc.SEQPAR24, [0, 10, 30]),
    }
    for name, text in sc.acceptance3_scenarios():
        golden["acc3-" + name] = record(lib, text, [0, 50, 100])
    for name, text in sc.EXTRA.items():
        golden["extra-" + name] = record(lib, text, [0, 5, 30])
    with open(os.path.join(HERE, "digests.json"), "w") as f:
        json.dump(golden, f, indent=1)
    print(f"wrote {len(golden)} entries")


if __name__ == "__main__":
    main()
