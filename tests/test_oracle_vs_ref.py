"""Validates the C restatement against the reference itself, compiled from its own sources
(oracle/_ref, `make -C oracle ref`): state for state and phase for phase, not only by digest.
Skipped where the reference library is absent."""
import numpy as np
import pytest

from oracle import oracle, shim
from tests import scenarios as sc


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint32 if a.dtype == np.float32 else np.uint64 if a.dtype == np.float64 else a.dtype)


@pytest.mark.parametrize("name", ["desk64", "closed-ped3", "ped5", "linear-regulation", "field-bigger-than-grid", "k16",
                                  "sparse-periodic", "sparse-closed", "sparse-field15", "field13-crowd"])
def test_phase_by_phase(ref_lib, name):
    text = sc.DESK64 if name == "desk64" else sc.EXTRA[name]
    ref = shim.Sim.from_scenario(ref_lib, text)
    cpu = oracle.OracleSim.from_scenario(text)
    np.testing.assert_array_equal(ref.centers(), cpu.centers())
    attrs_ref, attrs_cpu = ref.ped_attrs(), cpu.ped_attrs()
    for key in attrs_ref:
        np.testing.assert_array_equal(attrs_ref[key], attrs_cpu[key], err_msg=key)
    for tick in range(12 if ref.width * ref.height <= 8192 else 4):
        cap = ref.step_capture()
        probe = cpu.clone()
        probe.step(until_phase=4)
        np.testing.assert_array_equal(cap.decisions, probe.decisions())
        np.testing.assert_array_equal(cap.enroll_ids, probe.enroll_ids())
        np.testing.assert_array_equal(bits(cap.enroll_scores), bits(probe.enroll_scores()))
        np.testing.assert_array_equal(cap.winners, probe.winners())
        np.testing.assert_array_equal(cap.moved_from, probe.moved_from())
        np.testing.assert_array_equal(cap.moved_to, probe.moved_to())
        np.testing.assert_array_equal(cap.from_mask, probe.from_mask())
        np.testing.assert_array_equal(cap.to_mask, probe.to_mask())
        assert cap.moved == cpu.step()
        np.testing.assert_array_equal(ref.occupancy(), cpu.occupancy())
        for k in range(3):
            np.testing.assert_array_equal(bits(ref.image(k)), bits(cpu.image(k)))
        assert ref.digest() == cpu.digest()


def test_tables_match(ref_lib):
    for geom in [(7, 7), (5, 9), (21, 21)]:
        text = f"grid = 32x32\ndensity = 0.1\nfield_geometry = {geom[0]}x{geom[1]}\nfield_gain = 1.25\nfield_decay = -0.4\n"
        ref = shim.Sim.from_scenario(ref_lib, text)
        cpu = oracle.OracleSim.from_scenario(text)
        for kind in range(3):
            for orient in range(8):
                for sect in range(8):
                    d0, m0 = ref.plan_entries(kind, orient, sect)
                    d1, m1 = cpu.plan_entries(kind, orient, sect)
                    np.testing.assert_array_equal(d0, d1)
                    np.testing.assert_array_equal(bits(m0), bits(m1))


def test_static_fields_and_decide(ref_lib):
    anchors = [(0, 41, 41, 1.0, -0.02, 19, 10), (1, 7, 7, 2.0, -0.5, 4, 4), (1, 7, 7, 2.0, -0.5, 5, 4)]
    peds = [(3, 3, 0), (10, 10, 2), dict(x=15, y=6, goal=5, period=2, phase=1)]
    ref = shim.Sim.from_arrays(ref_lib, 20, 20, peds, closed=True)
    cpu = oracle.OracleSim.from_arrays(oracle.make_config(20, 20, closed=True), peds)
    ref.set_static_fields(anchors)
    cpu.set_static_fields(anchors)
    np.testing.assert_array_equal(bits(ref.image(-1)), bits(cpu.image(-1)))
    for i in range(3):
        d, s, _ = ref.decide(i)
        assert (d, s) == cpu.decide(i)
    for _ in range(10):
        ref.step()
        cpu.step()
    np.testing.assert_array_equal(ref.centers(), cpu.centers())


def test_seeding_stream(ref_lib):
    """mt19937_64 + uniform_int_distribution restated in C equals libstdc++'s: same centres,
    periods, phases and goals, including the sublattice-shuffle fallback (3x3 at rho 0.9)."""
    for name, text in sc.acceptance3_scenarios():
        ref = shim.Sim.from_scenario(ref_lib, text)
        cpu = oracle.OracleSim.from_scenario(text)
        np.testing.assert_array_equal(ref.centers(), cpu.centers(), err_msg=name)
        a, b = ref.ped_attrs(), cpu.ped_attrs()
        for key in a:
            np.testing.assert_array_equal(a[key], b[key], err_msg=f"{name} {key}")
