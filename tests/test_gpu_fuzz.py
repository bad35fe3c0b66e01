"""Seeded random scenarios against the oracle: grid extents (ragged, tiny, not a multiple of the 16-byte
staging group), field and pedestrian geometries, densities, chunk widths, boundaries, walk periods,
regulation, rebuild intervals — each through the engine's own choice of k-5 kernel and through a randomly
forced one (pair / field / list-walk / window / scatter kernel, row slabs, band-swapped pass), some with the
pedestrian kernels in position order, plain launches, or the tile stamps on.  Bit-exact."""
import os
import random

import numpy as np
import pytest

from oracle import oracle, shim
from tests import scenarios as sc  # noqa: F401

pytestmark = pytest.mark.gpu


def random_scenario(rng: random.Random):
    closed = rng.random() < 0.3
    fw, fh = rng.choice([(3, 3), (5, 5), (7, 7), (9, 9), (5, 9), (11, 7), (13, 13), (17, 15), (21, 21), (25, 31), (37, 37), (45, 29),
                         (7, 7), (7, 7), (61, 45), (77, 77), (9, 5), (15, 15), (19, 41)])
    pw, ph = rng.choice([(1, 1)] * 5 + [(3, 3), (3, 1), (1, 3), (5, 3)])
    big = rng.random() < 0.15
    w = rng.randint(max(6, pw + 2), 260 if big else 150)
    h = rng.randint(max(6, ph + 2), 190 if big else 110)
    area = pw * ph
    density = rng.choice([0.002, 0.01, 0.05, 0.15, 0.3, 0.5, 0.8]) / (1 if area == 1 else 1.6)
    lines = [f"grid = {w}x{h}", f"density = {density}", f"directions = {rng.choice(['uni', 'bi', 'four', 'eight'])}",
             f"field_geometry = {fw}x{fh}", f"pedestrian_geometry = {pw}x{ph}", f"chunk_k = {rng.choice([2, 4, 8, 8, 8, 16])}",
             f"seed = {rng.randint(1, 10 ** 6)}", f"rebuild_interval = {rng.choice([0, 3, 5, 50])}",
             f"walk_period = 1..{rng.choice([1, 1, 2, 3, 5])}"]
    if closed:
        lines.append("boundary = closed")
    if rng.random() < 0.25:
        lines += ["regulation = linear", f"density_radius = {rng.randint(0, 3)}"]
    if rng.random() < 0.3:
        lines += [f"field_gain = {rng.choice([0.5, 1.3, 2.0])}", f"field_decay = {rng.choice([-0.2, -0.37, -0.9])}",
                  f"goal_bias = {rng.choice([0.0, 0.35, 1.0, 2.5])}"]
    return "\n".join(lines) + "\n", (w, h, fw, fh, pw, ph)


def forced(rng: random.Random, dims):
    w, h, fw, fh, pw, ph = dims
    choices = [{}, {"SFC_K5_PATH": "field", "SFC_K5_FIELD_LAZY": rng.choice("01"), "SFC_K5_FIELD_NK": rng.choice("13")},
               {"SFC_K5_PATH": "scatter", "SFC_K5_EVENT_MAX": rng.choice(["0", "3", "100000"])},
               {"SFC_K5_PATH": "pairs", "SFC_K5_RED": rng.choice("01"), "SFC_K5_ACTIVE_LIST": rng.choice("01")},
               {"SFC_K5_PATH": "listwalk", "SFC_K5_ACTIVE_LIST": rng.choice("01")}, {"SFC_K5_PATH": "window"},
               {"SFC_GRAPH_TICKS": rng.choice(["1", "3", "7"])}]
    halo = max((fh - 1) // 2, 4 * ((ph - 1) // 2 + 1) + 3)
    if h >= 2 * (halo + 2) + 2 * halo:  # two slabs / bands of at least a halo, with room for both halos
        choices += [{"SFC_SLABS": "2"}, {"SFC_BANDS": "2"}]
    return rng.choice(choices)


CASES = int(os.environ.get("SFC_FUZZ_CASES", "60"))      # (a longer one-off hunt: SFC_FUZZ_CASES=1000 SFC_FUZZ_SEED=...)
SEED = int(os.environ.get("SFC_FUZZ_SEED", "9000"))


@pytest.mark.parametrize("case", range(CASES))
def test_random_scenarios_match_the_oracle(product_lib, monkeypatch, case):
    rng = random.Random(SEED + case)
    text, dims = random_scenario(rng)
    knobs = forced(rng, dims) if case % 2 else {}
    extras = random.Random(SEED + case + 10 ** 6)  # (a separate stream: the cases above keep their scenarios)
    if extras.random() < 0.3:
        knobs["SFC_PED_ORDER"] = "1"  # k-2 ... k-4 in position order
    if extras.random() < 0.2:
        knobs["SFC_CHAIN"] = "0"  # plain launches
    if extras.random() < 0.3 and knobs.get("SFC_K5_PATH") in (None, "pairs", "listwalk") and "SFC_SLABS" not in knobs and "SFC_BANDS" not in knobs:
        knobs["SFC_K5_ACTIVE_LIST"] = "1"  # tile stamps on: rebuilds may skip untouched tiles
    for k, v in knobs.items():
        monkeypatch.setenv(k, v)
    try:
        cpu = oracle.OracleSim.from_scenario(text)
    except Exception as exc:  # a density the footprint cannot be packed at: the reference rejects it too
        pytest.skip(f"oracle rejects the scenario: {exc}")
    try:
        gpu = shim.Sim.from_scenario(product_lib, text)
    except shim.ShimError as rejected:  # the scenario validator (scenario.cpp:134-170) — the C oracle is more lenient than it
        if shim.have_ref():
            with pytest.raises(shim.ShimError) as ref_rejected:
                shim.Sim.from_scenario(shim.load_ref(), text)
            assert (ref_rejected.value.kind, ref_rejected.value.message) == (rejected.kind, rejected.message)
        pytest.skip(f"rejected like the reference: {rejected}")
    label = f"case {case} {knobs} :: " + text.replace("\n", "; ")
    for ticks in (1, 2, 4, 6):
        np.testing.assert_array_equal(gpu.run(ticks), cpu.run(ticks), err_msg=label + " moved")
        np.testing.assert_array_equal(gpu.centers(), cpu.centers(), err_msg=label + f" tick {gpu.tick} centres")
        np.testing.assert_array_equal(gpu.occupancy(), cpu.occupancy(), err_msg=label + f" tick {gpu.tick} occupancy")
        for k in range(3):
            np.testing.assert_array_equal(gpu.image(k).view(np.uint32), cpu.image(k).view(np.uint32),
                                          err_msg=label + f" tick {gpu.tick} image {k}")
    assert gpu.digest() == cpu.digest(), label
