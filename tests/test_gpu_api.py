"""GPU tests through the reference-facing surfaces: the `socfield` Python module (the reference's
tests/python/test_smoke.py cases that need the engine) and socfield::Engine via the flat shim
(the unit cases of the reference's tests/unit/test_engine.cpp), each checked against the oracle."""
import numpy as np
import pytest

from oracle import oracle, shim
from tests import scenarios as sc
from paper_1803_04782_b200 import socfield as sf

pytestmark = pytest.mark.gpu

T = [(7, 7, 1.0, -0.5)] * 3


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint32 if a.dtype == np.float32 else np.uint64)


def pair(product_lib, w, h, peds, closed=False, **cfg):
    """The same hand-built population on the CUDA engine and on the oracle."""
    gpu = shim.Sim.from_arrays(product_lib, w, h, peds, closed=closed, cfg=shim.quiet_config(**cfg), templates=T)
    ocfg = {k: v for k, v in cfg.items() if k != "workers"}
    cpu = oracle.OracleSim.from_arrays(oracle.make_config(w, h, closed=closed, **ocfg), peds)
    return gpu, cpu


def same(gpu, cpu):
    np.testing.assert_array_equal(gpu.centers(), cpu.centers())
    np.testing.assert_array_equal(gpu.occupancy(), cpu.occupancy())
    for k in range(3):
        np.testing.assert_array_equal(bits(gpu.image(k)), bits(cpu.image(k)))
    assert gpu.tick == cpu.tick


# ---- reference tests/python/test_smoke.py ---------------------------------------------------

def test_smoke_seeding():
    cfg = sf.parse_scenario("grid = 32x32\ndensity = 0.5\nseed = 9\n")
    state = sf.seed_population(cfg)
    assert state.population == 512
    occ = state.occupancy()
    assert occ.shape == (32, 32) and (occ >= 0).sum() == 512
    img = state.image("recurrent-repulsive")
    assert img.shape == (32, 32, 8) and img.sum() > 0
    cpu = oracle.OracleSim.from_scenario("grid = 32x32\ndensity = 0.5\nseed = 9\n")
    np.testing.assert_array_equal(state.centers(), cpu.centers())
    for k, kind in enumerate(("dir-attractive", "dir-repulsive", "recurrent-repulsive")):
        np.testing.assert_array_equal(bits(state.image(kind)), bits(cpu.image(k)))


def test_smoke_engine_run_and_invariants():
    cfg = sf.parse_scenario("grid = 32x32\ndensity = 0.4\ndirections = four\nseed = 3\n")
    state = sf.seed_population(cfg)
    engine = sf.Engine(cfg, workers=2)
    metrics = engine.run(state, 10, mode="par")
    assert len(metrics) == 10 and state.tick == 10
    engine.verify_state(state)
    assert (state.occupancy() >= 0).sum() == state.population
    assert metrics[0].moved > 0
    assert engine.plan_fanout("recurrent-repulsive") == 7


def test_smoke_modes_identical_and_tick_equals_run():
    cfg = sf.parse_scenario("grid = 24x24\ndensity = 0.5\nseed = 21\n")
    a = sf.seed_population(cfg)
    b = a.copy()
    c = a.copy()
    sf.Engine(cfg, workers=1).run(a, 8, mode="seq")
    sf.Engine(cfg, workers=4).run(b, 8, mode="par")
    e = sf.Engine(cfg)
    for _ in range(8):
        e.tick(c)  # upload / one tick / download each call
    for other in (b, c):
        identical, diagnosis = sf.states_identical(a, other)
        assert identical, diagnosis


def test_resident_stepping_equals_run():
    cfg = sf.parse_scenario("grid = 40x28\ndensity = 0.3\nwalk_period = 1..3\nseed = 5\nrebuild_interval = 7\n")
    a = sf.seed_population(cfg)
    b = a.copy()
    sf.Engine(cfg).run(a, 23)
    e = sf.Engine(cfg)
    e.upload(b)
    m = e.step_resident(10) + e.step_resident(13, True)
    e.download(b)
    assert [x.tick for x in m] == list(range(23))
    identical, diagnosis = sf.states_identical(a, b)
    assert identical, diagnosis
    assert e.counters()["kernel_launches"] > 0


def test_one_engine_on_states_of_different_population():
    """Engine::run(SimState&, ...) takes any state of the engine's grid (engine.hpp:157-160).  A
    larger population, then a smaller one that fits the device arrays of the first, then the larger
    again: the replayed tick graph must follow the population size."""
    base = "grid = 48x40\ndirections = eight\nwalk_period = 1..2\nrebuild_interval = 6\n"
    texts = [base + "density = 0.5\nseed = 11\n", base + "density = 0.2\nseed = 12\n", base + "density = 0.45\nseed = 13\n"]
    engine = sf.Engine(sf.parse_scenario(texts[0]))
    for text in texts:
        state = sf.seed_population(sf.parse_scenario(text))
        cpu = oracle.OracleSim.from_scenario(text)
        for _ in range(2):
            moved = [m.moved for m in engine.run(state, 9)]
            np.testing.assert_array_equal(moved, cpu.run(9))
            np.testing.assert_array_equal(state.centers(), cpu.centers())
            np.testing.assert_array_equal(state.occupancy(), cpu.occupancy())
            for k, kind in enumerate(("dir-attractive", "dir-repulsive", "recurrent-repulsive")):
                np.testing.assert_array_equal(bits(state.image(kind)), bits(cpu.image(k)))


# ---- reference tests/unit/test_engine.cpp ---------------------------------------------------

def test_empty_grid_only_advances_the_counter(product_lib):
    gpu, cpu = pair(product_lib, 10, 10, [])
    before = gpu.images().copy()
    assert gpu.step() == 0 and gpu.tick == 1
    np.testing.assert_array_equal(gpu.images(), before)
    assert (gpu.occupancy() == -1).all()


def test_decide_cases(product_lib):
    gpu, cpu = pair(product_lib, 10, 10, [dict(x=5, y=5, goal=0, period=2)])
    gpu.tick = 1
    assert gpu.decide(0)[0] == -1                                   # walk gate (test_engine.cpp:128-137)
    gpu, cpu = pair(product_lib, 10, 10, [(5, 5, 0)], goal_bias=0.0)
    assert gpu.decide(0)[0] == -1                                   # no stimulus (:139-146)
    gpu, cpu = pair(product_lib, 10, 10, [(5, 5, 0)])
    d, s, cells = gpu.decide(0)
    assert (d, s, cells) == (0, 1.0, [(6, 5)])                      # goal bias (:148-159)
    gpu.step()
    assert gpu.centers().tolist() == [[6, 5]]
    gpu, cpu = pair(product_lib, 16, 16, [(8, 8, 0), (9, 8, 4)], goal_bias=0.0, weight_dir_attractive=0.0,
                    weight_dir_repulsive=0.0)
    d, s, _ = gpu.decide(0)
    assert d == 4 and s == cpu.decide(0)[1] and s == pytest.approx(np.exp(-0.5))  # (:161-178)


def test_vote_cases(product_lib):
    zero = dict(weight_static=0.0, weight_dir_attractive=0.0, weight_dir_repulsive=0.0, weight_recurrent=0.0)
    gpu, cpu = pair(product_lib, 8, 8, [(4, 4, 0), (6, 4, 4)], **zero)
    cap = gpu.step_capture()
    assert cap.winners[4 * 8 + 5] == 0 and (cap.enroll_ids.reshape(-1, 8)[4 * 8 + 5] >= 0).sum() == 2
    assert gpu.centers().tolist() == [[5, 4], [6, 4]]               # tie -> lower id (:192-213)
    gpu.verify()
    gpu, cpu = pair(product_lib, 8, 8, [(4, 4, 0), (6, 4, 4)], fault_invert_vote_tiebreak=1, **zero)
    gpu.step()
    assert gpu.centers().tolist() == [[4, 4], [5, 4]]               # fault hook (test_bench_cli.cpp:175-198)
    peds = [(4, 3, 0), (6, 4, 4), dict(x=5, y=3, goal=0, period=2, phase=1)]
    gpu, cpu = pair(product_lib, 8, 8, peds, **zero)
    cap = gpu.step_capture()
    assert cap.winners[4 * 8 + 5] == 1
    assert gpu.centers().tolist() == [[4, 3], [5, 4], [5, 3]]       # higher score beats lower id (:216-238)


def test_k4_log(product_lib):
    gpu, cpu = pair(product_lib, 8, 8, [(4, 4, 0)], goal_bias=0.0)
    cap = gpu.step_capture()
    assert (cap.moved_from == -1).all() and (cap.moved_to == -1).all()  # (:240-252)
    gpu, cpu = pair(product_lib, 8, 8, [(4, 4, 2)])
    cap = gpu.step_capture()
    assert cap.moved_from[4 * 8 + 4] == 0 and cap.moved_to[5 * 8 + 4] == 0  # (:254-266)
    assert gpu.centers().tolist() == [[4, 5]]
    gpu.verify()


@pytest.mark.parametrize("chunk", [2, 4, 8, 16])
def test_k5_one_move_equals_rerasterization(product_lib, chunk):
    gpu, cpu = pair(product_lib, 24, 24, [(10, 10, 1)], chunk_k=chunk)  # (:282-298)
    gpu.step()
    cpu.step()
    assert gpu.centers().tolist() == [[11, 11]]
    same(gpu, cpu)
    fresh = gpu.rebuild_images()
    np.testing.assert_array_equal(bits(fresh), bits(cpu.rebuild_images()))
    assert np.abs(gpu.images() - fresh).max() < 1e-6


def test_k5_no_movement_and_cross_chunk_agreement(product_lib):
    zero = dict(goal_bias=0.0, weight_static=0.0, weight_dir_attractive=0.0, weight_dir_repulsive=0.0,
                weight_recurrent=0.0)
    gpu, _ = pair(product_lib, 12, 12, [(4, 4, 0), (8, 8, 4)], **zero)
    before = gpu.images().copy()
    gpu.step()
    np.testing.assert_array_equal(bits(gpu.images()), bits(before))    # (:268-280)
    finals = []
    for chunk in (2, 4, 8, 16):                                         # (:300-327)
        gpu, cpu = pair(product_lib, 16, 16, [(4, 4, 0), (9, 9, 4), (12, 3, 2)], chunk_k=chunk)
        gpu.run(20)
        cpu.run(20)
        same(gpu, cpu)
        finals.append((gpu.centers(), gpu.images()))
    for c, img in finals[1:]:
        np.testing.assert_array_equal(c, finals[0][0])
        assert (np.abs(img - finals[0][1]) <= 1e-6 * (1 + np.abs(finals[0][1]))).all()


def test_field_larger_than_grid(product_lib):
    gpu, cpu = pair(product_lib, 8, 8, [(3, 3, 2)])                    # (:329-340)
    gpu.run(5)
    cpu.run(5)
    same(gpu, cpu)
    assert np.abs(gpu.images() - gpu.rebuild_images()).max() < 1e-5


def test_run_zero_ticks_and_rejections(product_lib):
    gpu, _ = pair(product_lib, 8, 8, [(4, 4, 0)])
    twin = gpu.clone()
    assert len(gpu.run(0)) == 0
    assert gpu.identical(twin)[0]                                       # (:342-350)
    occ = gpu.occupancy()
    occ[4, 4] = -1
    gpu.set_occupancy(occ)
    with pytest.raises(shim.ShimError) as e:                            # (:485-491)
        gpu.run(1)
    assert e.value.kind == "IntegrityError"
    gpu, _ = pair(product_lib, 8, 8, [(4, 4, 0)])
    occ = gpu.occupancy()
    occ[1, 1] = 0
    gpu.set_occupancy(occ)
    with pytest.raises(shim.ShimError, match="occupancy at su"):        # (:493-499)
        gpu.verify()
    with pytest.raises(shim.ShimError) as e:
        shim.Sim.from_arrays(product_lib, 8, 8, [], cfg=shim.quiet_config(chunk_k=3))
    assert e.value.kind == "ConfigError" and "chunk_k" in e.value.message


def test_rebuild_drift_is_an_integrity_error(product_lib):
    gpu, _ = pair(product_lib, 12, 12, [(4, 4, 0)], rebuild_interval=1)
    img = gpu.image(2)
    img[6, 6, 3] += 1.0
    gpu.set_image(2, img)
    with pytest.raises(shim.ShimError) as e:                            # (:442-451)
        gpu.step()
    assert e.value.kind == "IntegrityError"
    assert "recurrent-repulsive image drifted by 1.0" in e.value.message and "phase k-5" in e.value.message
    assert gpu.tick == 1  # the reference throws after the counter advanced, images left drifted
    assert gpu.image(2)[6, 6, 3] >= 1.0


def test_closed_boundary_and_wide_bodies(product_lib):
    gpu, cpu = pair(product_lib, 8, 8, [(7, 4, 0)], closed=True)
    assert gpu.decide(0)[0] == -1                                       # (:453-465)
    gpu, cpu = pair(product_lib, 8, 8, [(6, 4, 0)], closed=True)
    assert gpu.decide(0)[0] == 0
    gpu, cpu = pair(product_lib, 12, 12, [dict(x=5, y=5, goal=0, fw=3, fh=3)])
    gpu.step()
    assert gpu.centers().tolist() == [[6, 5]]                           # (:501-511)
    occ = gpu.occupancy()
    assert occ[4, 7] == 0 and occ[5, 4] == -1
    gpu.verify()
    d, s, cells = gpu.decide(0)
    assert cells == [(8, 4), (8, 5), (8, 6)] or d != 0


def test_conservation_speed_bound_and_gate(product_lib):
    text = "grid = 20x20\ndensity = 0.5\ndirections = bi\nseed = 5\n"   # (:379-408)
    gpu = shim.Sim.from_scenario(product_lib, text)
    attrs = gpu.ped_attrs()
    last = gpu.centers()
    for t in range(25):
        gpu.step()
        gpu.verify()
        now = gpu.centers()
        d = (now - last + 10) % 20 - 10
        assert np.abs(d).max() <= 1
        closed_gate = (t % attrs["period"]) != attrs["phase"]
        assert (d[closed_gate] == 0).all()
        last = now


# ---- static fields (openings / obstacles) ---------------------------------------------------

def test_static_fields_match_oracle(product_lib):
    """rasterize_static on the device, including a 41x41 field clipped by a closed boundary, two
    overlapping obstacle fields (list order matters in float), and the c1-style exit field larger
    than the room."""
    anchors = [(0, 41, 41, 1.0, -0.02, 19, 10), (1, 7, 7, 2.0, -0.5, 4, 4), (1, 7, 7, 2.0, -0.5, 5, 4),
               (1, 5, 9, 0.7, -0.3, 0, 19)]
    peds = [(3, 3, 0), (10, 10, 2), dict(x=15, y=6, goal=5, period=2, phase=1)]
    for closed in (True, False):
        gpu, cpu = pair(product_lib, 20, 20, peds, closed=closed)
        gpu.set_static_fields(anchors)
        cpu.set_static_fields(anchors)
        np.testing.assert_array_equal(bits(gpu.image(-1)), bits(cpu.image(-1)))
        for i in range(3):
            d, s, _ = gpu.decide(i)
            assert (d, s) == cpu.decide(i)
        gpu.run(12)
        cpu.run(12)
        same(gpu, cpu)


def test_c1_room_with_exit_field(product_lib):
    text = "grid = 200x200\nboundary = closed\ndensity = 0.0125\ndirections = uni\nseed = 42\nrebuild_interval = 50\n"
    gpu = shim.Sim.from_scenario(product_lib, text)
    cpu = oracle.OracleSim.from_scenario(text)
    exit_field = [(0, 399, 399, 1.0, -0.02, 199, 100)]
    gpu.set_static_fields(exit_field)
    cpu.set_static_fields(exit_field)
    np.testing.assert_array_equal(bits(gpu.image(-1)), bits(cpu.image(-1)))
    assert gpu.population == 500
    np.testing.assert_array_equal(gpu.run(60), cpu.run(60))
    same(gpu, cpu)


def test_python_set_static_fields():
    cfg = sf.parse_scenario("grid = 30x20\nboundary = closed\ndensity = 0.05\ndirections = uni\nseed = 2\n")
    state = sf.seed_population(cfg)
    state.set_static_fields([(sf.FieldSpec("omni-attractive", (59, 39), 1.0, -0.05), (29, 10)),
                             (sf.FieldSpec("omni-repulsive", (5, 5), 3.0, -0.5), (12, 9))])
    cpu = oracle.OracleSim.from_scenario("grid = 30x20\nboundary = closed\ndensity = 0.05\ndirections = uni\nseed = 2\n")
    cpu.set_static_fields([(0, 59, 39, 1.0, -0.05, 29, 10), (1, 5, 5, 3.0, -0.5, 12, 9)])
    np.testing.assert_array_equal(bits(state.image("static")), bits(cpu.image(-1)))
    sf.Engine(cfg).run(state, 30)
    cpu.run(30)
    np.testing.assert_array_equal(state.centers(), cpu.centers())


# ---- full-size property checks ---------------------------------------------------------------

def test_c2_full_size_properties(product_lib):
    """BASELINE config 2 at full size (2000x500, 20 000 pedestrians): bit-exact against the oracle
    for the first ticks, then size-independent properties over a longer horizon — conservation,
    structural validity, and the incremental images staying within float noise of a from-scratch
    rasterisation (no rebuild in between)."""
    text = ("grid = 2000x500\nboundary = periodic\ndensity = 0.02\ndirections = bi\nwalk_period = 1..3\n"
            "field_geometry = 7x7\nseed = 42\nrebuild_interval = 0\n")
    gpu = shim.Sim.from_scenario(product_lib, text)
    cpu = oracle.OracleSim.from_scenario(text)
    assert gpu.population == 20000
    np.testing.assert_array_equal(gpu.run(4), cpu.run(4))
    same(gpu, cpu)
    moved = gpu.run(300)
    assert moved.min() > 0 and moved.max() <= 20000
    gpu.verify()
    occ = gpu.occupancy()
    assert (occ >= 0).sum() == 20000 and len(np.unique(occ[occ >= 0])) == 20000
    c = gpu.centers()
    assert (occ[c[:, 1], c[:, 0]] == np.arange(20000)).all()
    assert np.abs(gpu.images() - gpu.rebuild_images()).max() < 1e-4


@pytest.mark.gpu
@pytest.mark.parametrize("text", [
    "grid = 96x64\ndensity = 0.3\ndirections = eight\nwalk_period = 1..3\nseed = 7\nrebuild_interval = 10\n",
    "grid = 70x50\nboundary = closed\ndensity = 0.1\ndirections = four\npedestrian_geometry = 3x3\nseed = 3\nrebuild_interval = 0\n",
])
def test_seed_resident_equals_host_seeding(text):
    """Engine.seed_resident (device-built occupancy and images, no host SimState) is bit-identical to
    upload(seed_population(cfg)) — scenario.cpp:392-429 — right after seeding and after 25 ticks."""
    cfg = sf.parse_scenario(text)
    host = sf.seed_population(cfg)
    a = sf.Engine(cfg)
    a.upload(host)
    b = sf.Engine(cfg)
    assert b.seed_resident(cfg) == host.population
    out = host.copy()
    for ticks in (0, 25):
        if ticks:
            a.step_resident(ticks)
            b.step_resident(ticks)
        a.download(host)
        b.download(out)
        assert np.array_equal(b.download_centers(), host.centers())
        assert np.array_equal(out.occupancy(), host.occupancy())
        for kind in ("dir-attractive", "dir-repulsive", "recurrent-repulsive"):
            assert np.array_equal(out.image(kind).view(np.uint32), host.image(kind).view(np.uint32)), kind


@pytest.mark.gpu
def test_c4_replica_sparse_paths_agree(monkeypatch):
    """BASELINE config 4 (32768^2, 1M pedestrians) at 1/64 of the area, same density, geometry and
    fields, seeded on the device.  The sparse crowd switches k-5 to the active-tile list + window
    kernel; a second engine forced onto the every-tile scatter kernel must end in the identical state
    (positions, occupancy, f32 images bit for bit) after 60 ticks and one rebuild, and the run keeps
    the model's invariants: population conserved, one su per pedestrian, Chebyshev speed <= 1."""
    text = ("grid = 4096x4096\ndensity = 0.000931322574615478515625\ndirections = eight\nfield_geometry = 7x7\n"
            "seed = 42\nrebuild_interval = 50\n")
    cfg = sf.parse_scenario(text)
    a = sf.Engine(cfg)                      # by density: window kernel over the active-tile list
    monkeypatch.setenv("SFC_K5_PATH", "scatter")
    monkeypatch.setenv("SFC_K5_ACTIVE_LIST", "0")
    b = sf.Engine(cfg)                      # every tile, scatter + dense gather
    n = a.seed_resident(cfg)
    assert n == b.seed_resident(cfg) == 15625
    prev = a.download_centers()
    for _ in range(6):
        ma = a.step_resident(10)
        mb = b.step_resident(10)
        assert [m.moved for m in ma] == [m.moved for m in mb]
        ca, cb = a.download_centers(), b.download_centers()
        assert np.array_equal(ca, cb)
        d = np.abs(ca.astype(np.int64) - prev.astype(np.int64))
        d = np.minimum(d, 4096 - d)         # periodic
        assert d.max() <= 10                # <= 1 su per tick
        prev = ca
    sa = sf.seed_population(cfg)            # download target (a host SimState of the right shape)
    a.download(sa)
    sb = sa.copy()
    b.download(sb)
    occ = sa.occupancy()
    assert (occ >= 0).sum() == n and len(np.unique(occ[occ >= 0])) == n
    assert np.array_equal(occ, sb.occupancy())
    assert np.array_equal(occ[prev[:, 1], prev[:, 0]], np.arange(n))
    for kind in ("dir-attractive", "dir-repulsive", "recurrent-repulsive"):
        assert np.array_equal(sa.image(kind).view(np.uint32), sb.image(kind).view(np.uint32)), kind


@pytest.mark.gpu
@pytest.mark.parametrize("path", ["default", "window", "scatter", "scatter-gather-all"])
def test_kinds_with_different_field_geometries(product_lib, monkeypatch, path):
    """The Engine takes one FieldSpec per kind (engine.hpp:144-145) and they need not share a
    geometry — only the scenario format ties them together.  Kinds with different supports cannot
    share contributor lists (no list walk, no combined gating word): every k-5 path must fall back to
    its general form and still match the oracle bit for bit."""
    if path != "default":
        monkeypatch.setenv("SFC_K5_PATH", path.split("-")[0])
    if path == "scatter-gather-all":
        monkeypatch.setenv("SFC_K5_EVENT_MAX", "0")
    templates = [(7, 7, 1.0, -0.5), (5, 9, 1.3, -0.4), (9, 5, 0.8, -0.6)]
    rng = np.random.default_rng(5)
    w, h = 61, 43
    cells = rng.choice(w * h, size=260, replace=False)
    peds = [dict(x=int(c % w), y=int(c // w), goal=int(rng.integers(8)), period=int(p), phase=int(rng.integers(p)))
            for c, p in zip(cells, rng.integers(1, 4, size=260))]
    cfg = dict(goal_bias=1.0, rebuild_interval=7)
    gpu = shim.Sim.from_arrays(product_lib, w, h, peds, cfg=shim.quiet_config(**cfg), templates=templates)
    cpu = oracle.OracleSim.from_arrays(oracle.make_config(w, h, templates=templates, **cfg), peds)
    total = 0
    for _ in range(5):
        moved = cpu.run(6)
        np.testing.assert_array_equal(gpu.run(6), moved)
        total += int(moved.sum())
        same(gpu, cpu)
        for k in range(3):
            np.testing.assert_array_equal(bits(gpu.image(k)), bits(cpu.image(k)))
    assert total > 500  # the crowd really moves


@pytest.mark.gpu
def test_one_run_across_the_stamp_period(monkeypatch):
    """A single run longer than the 65535-tick period of the active-tile stamps: without the periodic
    erase a tile last listed exactly one period earlier would look already listed and be skipped.
    The list-driven window path must end where the every-tile list walk ends."""
    text = "grid = 96x64\ndensity = 0.004\ndirections = eight\nseed = 9\nrebuild_interval = 0\n"
    cfg = sf.parse_scenario(text)
    a_state, b_state = sf.seed_population(cfg), sf.seed_population(cfg)
    monkeypatch.setenv("SFC_K5_PATH", "window")
    a = sf.Engine(cfg)
    monkeypatch.setenv("SFC_K5_PATH", "listwalk")
    monkeypatch.setenv("SFC_K5_ACTIVE_LIST", "0")
    b = sf.Engine(cfg)
    ticks = 65535 + 40
    ma = a.run(a_state, ticks)
    mb = b.run(b_state, ticks)
    assert [m.moved for m in ma[-200:]] == [m.moved for m in mb[-200:]]
    same, why = sf.states_identical(a_state, b_state)
    assert same, why


@pytest.mark.parametrize("name,bands", [("desk64", 2), ("desk64", 3), ("closed-four", 2), ("linear-regulation", 2), ("wide-ragged", 3),
                                        ("field21", 2), ("ped5", 2), ("k16", 2), ("field35", 2), ("d0.9-eight-ped1", 4),
                                        ("field13-crowd", 2)])  # (13 x 13 in a crowd: scatter kernel handing tiles to the dense kernel, per band)
def test_band_swapped_pass_equals_undivided_grid(product_lib, monkeypatch, name, bands):
    """A state larger than device memory streams through the device in row bands, the host SimState
    being the backing store (sfc_band_run: the paper's divide-and-conquer as a band pass; reference
    accumulator.hpp:68-83, bench.cpp:14-24).  Forced here on small grids with SFC_BANDS: bit-identical
    to the oracle — i.e. to the undivided grid — across rebuilds, for every k-5 kernel family."""
    monkeypatch.setenv("SFC_BANDS", str(bands))
    text = sc.DESK64 if name == "desk64" else sc.EXTRA.get(name) or dict(sc.acceptance3_scenarios())[name]
    gpu = shim.Sim.from_scenario(product_lib, text)
    cpu = oracle.OracleSim.from_scenario(text)
    for chunk in (1, 7, 14):
        np.testing.assert_array_equal(gpu.run(chunk), cpu.run(chunk), err_msg=f"{name} x{bands} moved")
        assert gpu.tick == cpu.tick
        np.testing.assert_array_equal(gpu.centers(), cpu.centers(), err_msg=f"{name} x{bands} tick {gpu.tick} centres")
        np.testing.assert_array_equal(gpu.occupancy(), cpu.occupancy(), err_msg=f"{name} x{bands} tick {gpu.tick} occupancy")
        for k in range(3):
            np.testing.assert_array_equal(gpu.image(k).view(np.uint32), cpu.image(k).view(np.uint32), err_msg=f"{name} x{bands} image {k}")
    gpu.verify()


def test_band_plan_counts_bands_from_device_memory():
    """sfc_band_plan: 1 band when the state fits, more as the budget shrinks, -1 when a band cannot be cut thinner
    than its halo (134 B per resident su)."""
    import ctypes

    from paper_1803_04782_b200 import build

    lib = ctypes.CDLL(build.build_all(force=False, verbose=False)["cuda"])
    lib.sfc_band_plan.restype = ctypes.c_int
    lib.sfc_band_plan.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int64, ctypes.c_int64, ctypes.c_int]
    state = 135 * 49152 * 49152  # a 49152^2 grid: 326 GB resident, beyond one B200
    assert lib.sfc_band_plan(49152, 49152, 4, 1_000_000, 2 * state, 0) == 1
    assert lib.sfc_band_plan(49152, 49152, 4, 1_000_000, 170 << 30, 0) == 2
    assert lib.sfc_band_plan(49152, 49152, 4, 1_000_000, 60 << 30, 0) == 6
    assert lib.sfc_band_plan(64, 64, 40, 100, 1 << 20, 0) == -1


def test_run_bench_sweeps_like_the_reference():
    """run_bench on the CUDA engine (reference bench.cpp:65-124; cases of test_bench_cli.cpp:69-141):
    cross-product row counting, a failing combination recorded while the sweep continues, one row
    per walk period, exclusive axes; the report keeps the reference's header and columns."""
    base = sf.parse_scenario("grid = 16x16\ndensity = 0.3\n")
    rows, csv = sf.run_bench(base, grids=[(12, 12), (16, 16)], densities=[0.2, 0.4], directions=["uni"], ticks=2, repeats=2,
                             warmup=False, gpu_columns=False)
    assert len(rows) == 4
    for r in rows:
        assert r["status"] == "ok" and r["repeats"] == 2 and r["min_ms"] <= r["mean_ms"] <= r["max_ms"] and r["device_mean_ms"] > 0
    lines = csv.strip().splitlines()
    assert len(lines) == 5
    assert lines[0] == ("grid,density,directions,field_geometry,pedestrian_geometry,walk_period_max,population,sf,ticks,repeats,"
                        "mean_ms,min_ms,max_ms,status")
    assert [r["grid"] for r in rows] == [(12, 12), (12, 12), (16, 16), (16, 16)] and [r["density"] for r in rows] == [0.2, 0.4, 0.2, 0.4]

    base = sf.parse_scenario("grid = 10x10\n")
    rows, _ = sf.run_bench(base, densities=[0.9, 0.3], pedestrian_geometries=[(3, 3)], ticks=1, repeats=1, warmup=False)
    assert len(rows) == 2 and rows[0]["status"].startswith("error:") and rows[1]["status"] == "ok"
    assert rows[1]["field_geometry"] == (21, 21)  # joint geometry: fields scale with the body

    base = sf.parse_scenario("grid = 12x12\ndensity = 0.4\n")
    rows, csv = sf.run_bench(base, walk_period_maxes=[1, 3, 5, 7, 9, 11], ticks=1, repeats=1, warmup=False)
    assert [r["walk_period_max"] for r in rows] == [1, 3, 5, 7, 9, 11] and all(r["status"] == "ok" for r in rows)
    assert csv.splitlines()[0].endswith("device_mean_ms,ped_steps_per_s,su_updates_per_s,status")

    with pytest.raises(sf.ConfigError):
        sf.run_bench(base, field_ratios=[1], pedestrian_geometries=[(1, 1)])
    rows, _ = sf.run_bench(base, field_ratios=[1, 3], ticks=1, repeats=1, warmup=False)
    assert [r["field_geometry"] for r in rows] == [(7, 7), (21, 21)] and [r["sf"] for r in rows] == [7, 64]


def test_validate_tool_exit_codes(tmp_path, capsys):
    """`validate` (reference cmd_validate, cli.cpp:79-140; cases of test_bench_cli.cpp:175-198): two execution
    strategies of the engine in lockstep, compared on the device — identical runs exit 0, the injected vote
    tie-break fault is caught (exit 4), a malformed scenario exits 1, an impossible one 2."""
    from paper_1803_04782_b200 import validate

    desk = tmp_path / "desk.scn"
    desk.write_text(sc.variant(sc.DESK64, ticks=12))
    assert validate.main([str(desk)]) == 0
    assert validate.main([str(desk), "--variant", "SFC_K5_PATH=scatter,SFC_K5_EVENT_MAX=3"]) == 0
    assert validate.main([str(desk), "--variant", "SFC_K5_PATH=field", "--every", "4"]) == 0
    assert validate.main([str(desk), "--slabs", "2", "--every", "6"]) == 0
    assert validate.main([str(desk), "--bands", "2", "--every", "6"]) == 0
    assert "identical over 12 ticks" in capsys.readouterr().out
    assert validate.main([str(desk), "--ticks", "40", "--inject-tiebreak-fault"]) == 4
    assert "divergence at tick" in capsys.readouterr().err
    bad = tmp_path / "bad.scn"
    bad.write_text("grid = banana\n")
    assert validate.main([str(bad)]) == 1
    dense = tmp_path / "dense.scn"
    dense.write_text("grid = 10x10\ndensity = 1.5\n")
    assert validate.main([str(dense)]) == 2
    assert validate.main([str(tmp_path / "absent.scn")]) == 1

