"""BASELINE.json configs 1-5 on the CUDA engine at (or shaped like) their stated parameters, against
digests recorded from the UNMODIFIED reference (tests/golden/baseline_shaped.json, written by
tests/golden/make_golden.py --big): c1 over its full 1000 ticks, c2 over 100, the 35 x 35 fields of
c3, the c4 crowd (7 x 7 fields, one pedestrian per ~1000 su, active-tile list) on 4096 x 4096, and
c5's 77 x 77 fields together with linear regulation and obstacle fields.

The digest of the resident state is computed ON THE DEVICE (sfc_digest: exact FNV-1a, no host copy);
if one ever differs, the CPU oracle is run alongside to name the first differing array.
"""
import json
import os

import numpy as np
import pytest

from oracle import oracle
from paper_1803_04782_b200 import socfield as sf
from tests import scenarios as sc

pytestmark = pytest.mark.gpu

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "baseline_shaped.json")))
KINDS = ("omni-attractive", "omni-repulsive")


def bits(a):
    return np.ascontiguousarray(a).view(np.uint32)


def seeded(spec):
    cfg = sf.parse_scenario(spec["text"])
    state = sf.seed_population(cfg)
    if spec["static"]:
        state.set_static_fields([(sf.FieldSpec(KINDS[k], (w, h), gain, decay), (x, y)) for k, w, h, gain, decay, x, y in spec["static"]])
    return cfg, state


def explain(spec, engine, state, tick):
    """Digest mismatch: run the oracle to the same tick and name the first differing array."""
    oracle.OracleSim.set_threads(os.cpu_count() or 1)
    cpu = oracle.OracleSim.from_scenario(spec["text"])
    if spec["static"]:
        cpu.set_static_fields(spec["static"])
    cpu.run(tick)
    engine.download(state)
    np.testing.assert_array_equal(state.centers(), cpu.centers(), err_msg=f"tick {tick} centres")
    np.testing.assert_array_equal(state.occupancy(), cpu.occupancy(), err_msg=f"tick {tick} occupancy")
    for k, kind in enumerate(("dir-attractive", "dir-repulsive", "recurrent-repulsive")):
        np.testing.assert_array_equal(bits(state.image(kind)), bits(cpu.image(k)), err_msg=f"tick {tick} image {kind}")


@pytest.mark.parametrize("name", sorted(sc.BASELINE_SHAPED))
def test_baseline_config_against_reference_digests(name):
    spec, g = sc.BASELINE_SHAPED[name], GOLDEN[name]
    assert g["scenario"] == spec["text"] and g["static_fields"] == [list(a) for a in spec["static"]]
    cfg, state = seeded(spec)
    assert state.population == g["population"]
    engine = sf.Engine(cfg)
    engine.upload(state)
    last = 0
    for tick, digest in g["digests"]:
        engine.step_resident(tick - last)
        last = tick
        if f"{engine.digest():#018x}" != digest:
            explain(spec, engine, state, tick)
            pytest.fail(f"{name}: digest differs from the reference's at tick {tick} but the arrays match the oracle")
    engine.download(state)
    engine.verify_state(state)
    assert state.tick == last


@pytest.mark.parametrize("path", ["window", "listwalk", "scatter", "pairs-plain"])
def test_c4_shaped_every_small_field_path(monkeypatch, path):
    """The c4 crowd through every k-5 formulation that can take 7 x 7 fields (the default, the pair
    kernel over the active-tile list with float reductions, is the test above): window kernel + hand-off,
    list walk and scatter driven from the list, the pair kernel with plain read-modify-writes."""
    if path == "pairs-plain":
        monkeypatch.setenv("SFC_K5_PATH", "pairs")
        monkeypatch.setenv("SFC_K5_RED", "0")
    else:
        monkeypatch.setenv("SFC_K5_PATH", path)
        monkeypatch.setenv("SFC_K5_ACTIVE_LIST", "1")
    spec, g = sc.BASELINE_SHAPED["c4-4096"], GOLDEN["c4-4096"]
    cfg, state = seeded(spec)
    engine = sf.Engine(cfg)
    engine.upload(state)
    tick, digest = g["digests"][1]  # past the first rebuild
    engine.step_resident(tick)
    assert f"{engine.digest():#018x}" == digest


def test_device_digest_and_identity(product_lib):
    """sfc_digest equals the host-side FNV-1a of the downloaded state on grids whose byte stream
    spans many digest runs and ragged run ends; sfc_compare reports the reference's first
    difference (states_identical wording)."""
    from oracle import shim

    for text in (sc.DESK64, sc.EXTRA["wide-ragged"], sc.EXTRA["sparse-periodic"], "grid = 9x7\ndensity = 0.4\ndirections = uni\nseed = 2\n"):
        cfg = sf.parse_scenario(text)
        state = sf.seed_population(cfg)
        a, b = sf.Engine(cfg), sf.Engine(cfg)
        a.upload(state)
        b.upload(state)
        cpu = oracle.OracleSim.from_scenario(text)
        assert a.digest() == cpu.digest()
        a.step_resident(7)
        cpu.run(7)
        assert a.digest() == cpu.digest()
        same, why = a.identical_to(b)
        assert not same and why == "tick counter differs"
        b.step_resident(7)
        assert a.identical_to(b) == (True, "")
        a.download(state)
        if state.occupancy().size <= 4096:  # (pure-Python FNV-1a: small states only)
            assert shim.fnv1a_digest(state.occupancy(), [state.image(k) for k in ("dir-attractive", "dir-repulsive", "recurrent-repulsive")],
                                     state.centers()) == a.digest()
    # a difference in an image, then in the occupancy: reported in the reference's order
    cfg = sf.parse_scenario(sc.DESK64)
    state = sf.seed_population(cfg)
    other = state.copy()
    a, b = sf.Engine(cfg), sf.Engine(cfg)
    a.upload(state)
    img = other.image("dir-repulsive").copy()
    img[10, 20, 3] += 1.0
    other.set_image("dir-repulsive", img)
    b.upload(other)
    same, why = a.identical_to(b)
    assert not same and why.startswith("dir-repulsive image at su (20,10) sect 3:"), why
