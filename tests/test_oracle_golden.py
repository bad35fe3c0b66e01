"""Pins the CPU oracle (oracle/socfield_oracle.c) to the reference's golden vectors.

tests/golden/digests.json holds FNV-1a state digests recorded from the unmodified reference
(tests/golden/make_golden.py).  The C restatement must reproduce every one of them from the
scenario text alone — which exercises its seeding stream (mt19937_64 + libstdc++
uniform_int_distribution + shuffle), table construction, all five phases, the id-ordered float
rebuild and the K-slot summation order.
"""
import json
import os

import numpy as np
import pytest

from oracle import oracle

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "digests.json")))


@pytest.mark.parametrize("name", sorted(GOLDEN))
def test_oracle_reproduces_golden_digest(name):
    g = GOLDEN[name]
    sim = oracle.OracleSim.from_scenario(g["scenario"])
    assert sim.population == g["population"]
    last = 0
    for tick, digest in g["digests"]:
        sim.run(tick - last)
        last = tick
        assert f"{sim.digest():#018x}" == digest, f"{name} at tick {tick}"


BIG = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "baseline_shaped.json")))


@pytest.mark.parametrize("name", sorted(BIG))
def test_oracle_reproduces_baseline_shaped_digests(name):
    """BASELINE configs 1-5 at / shaped like their stated parameters (tests/scenarios.py
    BASELINE_SHAPED): c1 over 1000 ticks, c2 over 100, 35 x 35 fields, the c4 crowd on 4096^2,
    77 x 77 fields with linear regulation and obstacle fields — digests recorded from the unmodified
    reference.  The oracle's k-5 runs on every core here (static su partition, like the reference's
    parallel_for: the result does not depend on the worker count)."""
    g = BIG[name]
    oracle.OracleSim.set_threads(os.cpu_count() or 1)
    try:
        sim = oracle.OracleSim.from_scenario(g["scenario"])
        if g["static_fields"]:
            sim.set_static_fields([tuple(a) for a in g["static_fields"]])
        assert sim.population == g["population"]
        last = 0
        for tick, digest in g["digests"]:
            sim.run(tick - last)
            last = tick
            assert f"{sim.digest():#018x}" == digest, f"{name} at tick {tick}"
    finally:
        oracle.OracleSim.set_threads(1)


def test_oracle_k5_does_not_depend_on_the_thread_count():
    text = "grid = 96x80\ndensity = 0.3\ndirections = eight\nwalk_period = 1..2\nseed = 6\nrebuild_interval = 5\n"
    a = oracle.OracleSim.from_scenario(text)
    b = oracle.OracleSim.from_scenario(text)
    a.run(12)
    oracle.OracleSim.set_threads(5)
    try:
        b.run(12)
    finally:
        oracle.OracleSim.set_threads(1)
    assert a.digest() == b.digest()


def test_survey_vectors_are_in_the_fixture():
    """The five digests quoted in SURVEY.md 8(c) (captured independently of this repo)."""
    desk = dict(GOLDEN["desk64"]["digests"])
    assert desk[0] == "0xf28f22891b930483"
    assert desk[1] == "0xcfb64229b2b639f7"
    assert desk[10] == "0x4e5b561095510673"
    assert desk[100] == "0x479c4a4ca39c6e2a"
    assert dict(GOLDEN["seqpar24"]["digests"])[30] == "0x0d0d96dd2ede094f"
    assert GOLDEN["desk64"]["population"] == 2048 and GOLDEN["seqpar24"]["population"] == 230


def test_survey_centres():
    sim = oracle.OracleSim.from_scenario(GOLDEN["desk64"]["scenario"])
    sim.run(1)
    assert sim.centers()[:3].tolist() == [[49, 40], [48, 8], [58, 7]]
    sim.run(99)
    assert sim.centers()[:3].tolist() == [[12, 56], [60, 19], [56, 31]]


# ---- known-answer tests restated from the reference's unit tests ---------------------------

def test_sort8_known_answers():
    """test_engine.cpp:62-67 fixed vectors + :69-82 zero-one principle."""
    L = oracle.lib()
    import ctypes as C

    def sort8(v):
        a = (C.c_double * 8)(*v)
        o = (C.c_int32 * 8)()
        L.so_sort8_desc(a, o)
        return list(o)

    assert sort8([0] * 8) == list(range(8))
    assert sort8([8, 7, 6, 5, 4, 3, 2, 1]) == list(range(8))
    assert sort8([1, 2, 3, 4, 5, 6, 7, 8]) == [7, 6, 5, 4, 3, 2, 1, 0]
    assert sort8([0, 5, 0, 5, 0, 0, 0, 0]) == [1, 3, 0, 2, 4, 5, 6, 7]
    for bits in range(256):
        s = [(bits >> i) & 1 for i in range(8)]
        order = sort8(s)
        assert order == sorted(range(8), key=lambda i: (-s[i], i))
    rng = np.random.default_rng(42)
    for trial in range(2000):
        s = rng.uniform(-1, 1, 8) if trial % 2 else rng.integers(0, 4, 8).astype(float)
        assert sort8(list(s)) == sorted(range(8), key=lambda i: (-s[i], i))


def test_sect_index_known_answers():
    """test_smoke.py:23-27 and the wedge edges of fields.cpp:54-60."""
    L = oracle.lib()
    assert L.so_sect_index(1.0, 0.0) == 0
    assert L.so_sect_index(1.0, 1.0) == 1
    assert L.so_sect_index(3.0, 2.0) == 1
    assert L.so_sect_index(0.0, 0.0) == -1
    assert L.so_sect_index(-1.0, 0.0) == 4
    assert L.so_sect_index(0.0, -1.0) == 6
    assert L.so_sect_index(1.0, -1.0) == 7


def test_multi_step_sum_matches_one_step():
    """acceptance criterion 2 / test_smoke.py:30-38: regrouping, not a different sum."""
    L = oracle.lib()
    rng = np.random.default_rng(7)
    terms = rng.uniform(-5, 5, 481)
    one = L.so_one_step_sum(terms.ctypes.data, terms.size)
    for k in (2, 4, 8, 16):
        assert L.so_multi_step_sum(terms.ctypes.data, terms.size, k) == pytest.approx(one, rel=1e-9, abs=1e-9)
    ints = np.arange(1, 100, dtype=np.float64)
    for k in (2, 4, 8, 16):
        assert L.so_multi_step_sum(ints.ctypes.data, ints.size, k) == 4950.0


def test_write_plan_fanout_7x7():
    """test_smoke.py:41-46: 7x7 recurrent field: fan-out 7, 48 contributors."""
    cfg = oracle.make_config(16, 16)
    sim = oracle.OracleSim.from_arrays(cfg, [])
    lens = [len(sim.plan_entries(2, 0, s)[0]) for s in range(8)]
    assert lens == [5, 7, 5, 7, 5, 7, 5, 7] and sum(lens) == 48


def test_decide_and_vote_known_answers():
    """test_engine.cpp:128-238 restated on the oracle."""
    # goal bias moves a lone pedestrian toward +x
    sim = oracle.OracleSim.from_arrays(oracle.make_config(10, 10), [(5, 5, 0)])
    assert sim.decide(0) == (0, 1.0)
    sim.step()
    assert sim.centers().tolist() == [[6, 5]]
    # walk gate closed on off-phase ticks
    sim = oracle.OracleSim.from_arrays(oracle.make_config(10, 10), [dict(x=5, y=5, goal=0, period=2)])
    sim.tick = 1
    assert sim.decide(0)[0] == -1
    # no stimulus means Still
    sim = oracle.OracleSim.from_arrays(oracle.make_config(10, 10, goal_bias=0.0), [(5, 5, 0)])
    assert sim.decide(0)[0] == -1
    # a repulsive-only neighbour due +x pushes toward -x with score exp(-0.5)
    cfg = oracle.make_config(16, 16, goal_bias=0.0, weight_dir_attractive=0.0, weight_dir_repulsive=0.0)
    sim = oracle.OracleSim.from_arrays(cfg, [(8, 8, 0), (9, 8, 4)])
    d, s = sim.decide(0)
    assert d == 4 and s == pytest.approx(np.exp(-0.5))
    # exact tie -> lower id wins, one moves
    cfg = oracle.make_config(8, 8, weight_static=0, weight_dir_attractive=0, weight_dir_repulsive=0, weight_recurrent=0)
    sim = oracle.OracleSim.from_arrays(cfg, [(4, 4, 0), (6, 4, 4)])
    sim.step()
    assert sim.centers().tolist() == [[5, 4], [6, 4]]
    # fault hook inverts the tie-break
    cfg.fault_invert_vote_tiebreak = 1
    sim = oracle.OracleSim.from_arrays(cfg, [(4, 4, 0), (6, 4, 4)])
    sim.step()
    assert sim.centers().tolist() == [[4, 4], [5, 4]]
    # higher score beats lower id
    cfg.fault_invert_vote_tiebreak = 0
    sim = oracle.OracleSim.from_arrays(cfg, [(4, 3, 0), (6, 4, 4), dict(x=5, y=3, goal=0, period=2, phase=1)])
    sim.step()
    assert sim.centers().tolist() == [[4, 3], [5, 4], [5, 3]]


def test_k5_matches_rerasterization():
    """test_engine.cpp:282-340: incremental write-back vs from-scratch images, all chunk widths,
    including the 7x7 field on an 8x8 torus that wraps onto itself."""
    for k in (2, 4, 8, 16):
        sim = oracle.OracleSim.from_arrays(oracle.make_config(24, 24, chunk_k=k), [(10, 10, 1)])
        sim.step()
        assert sim.centers().tolist() == [[11, 11]]
        assert np.abs(sim.images() - sim.rebuild_images()).max() < 1e-6
    sim = oracle.OracleSim.from_arrays(oracle.make_config(8, 8), [(3, 3, 2)])
    sim.run(5)
    assert np.abs(sim.images() - sim.rebuild_images()).max() < 1e-5


def test_rebuild_drift_raises():
    """test_engine.cpp:442-451."""
    sim = oracle.OracleSim.from_arrays(oracle.make_config(12, 12, rebuild_interval=1), [(4, 4, 0)])
    sim.image(2)[6, 6, 3] += 1.0
    with pytest.raises(oracle.OracleError) as e:
        sim.step()
    assert e.value.phase == 5


def test_closed_boundary_and_3x3():
    """test_engine.cpp:453-483, 501-511."""
    sim = oracle.OracleSim.from_arrays(oracle.make_config(8, 8, closed=True), [(7, 4, 0)])
    assert sim.decide(0)[0] == -1
    sim = oracle.OracleSim.from_arrays(oracle.make_config(8, 8, closed=True), [(6, 4, 0)])
    assert sim.decide(0)[0] == 0
    sim = oracle.OracleSim.from_arrays(oracle.make_config(12, 12), [dict(x=5, y=5, goal=0, fw=3, fh=3)])
    sim.step()
    assert sim.centers().tolist() == [[6, 5]]
    occ = sim.occupancy()
    assert occ[4, 7] == 0 and occ[5, 4] == -1
    sim.verify()


def test_inconsistent_state_rejected():
    """test_engine.cpp:485-499."""
    sim = oracle.OracleSim.from_arrays(oracle.make_config(8, 8), [(4, 4, 0)])
    sim.occupancy()[4, 4] = -1
    with pytest.raises(oracle.OracleError):
        sim.run(1)
