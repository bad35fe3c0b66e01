"""GPU parity: the CUDA engine against the CPU oracle on identical scenarios and seeds.

Every comparison is BIT-EXACT (integers: occupancy, centres, decisions, vote winners, movement
log; floats compared by bit pattern: decision scores in f64, strength images in f32) — stronger
than the rtol 1e-5 the north star allows for field values.  The engine is reached through the
flat-C shim compiled against the product's host mirror, i.e. through socfield::Engine and the
C ABI underneath; the checker is the C oracle (oracle/socfield_oracle.c), cross-checked against
the compiled reference (oracle/_ref) when that library travelled with the snapshot.
"""
import json
import os

import numpy as np
import pytest

from oracle import oracle, shim
from tests import scenarios as sc

pytestmark = pytest.mark.gpu

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "digests.json")))


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint32 if a.dtype == np.float32 else np.uint64 if a.dtype == np.float64 else a.dtype)


def assert_state_equal(gpu: shim.Sim, cpu: oracle.OracleSim, label=""):
    assert gpu.tick == cpu.tick, label
    np.testing.assert_array_equal(gpu.centers(), cpu.centers(), err_msg=f"{label} centres")
    np.testing.assert_array_equal(gpu.occupancy(), cpu.occupancy(), err_msg=f"{label} occupancy")
    for k in range(3):
        np.testing.assert_array_equal(bits(gpu.image(k)), bits(cpu.image(k)), err_msg=f"{label} image {k}")
    assert gpu.digest() == cpu.digest(), label


@pytest.mark.parametrize("name", ["desk64", "seqpar24"])
def test_golden_digests(product_lib, name):
    """Free run from the seeded state reproduces the reference's recorded digests — through two
    id-ordered float rebuilds for desk64 (ticks 50 and 100)."""
    g = GOLDEN[name]
    sim = shim.Sim.from_scenario(product_lib, g["scenario"])
    assert sim.population == g["population"]
    last = 0
    for tick, digest in g["digests"]:
        sim.run(tick - last)
        last = tick
        assert f"{sim.digest():#018x}" == digest, f"{name} tick {tick}"


@pytest.mark.parametrize("name,text", sc.acceptance3_scenarios())
def test_acceptance3_free_run(product_lib, name, text):
    """Acceptance criterion 3's 24 scenarios (64x64; rho .1/.5/.9; 4 direction sets; 1x1 and 3x3
    pedestrians; rebuild every 50), 100 ticks: state identical to the oracle every 10 ticks."""
    gpu = shim.Sim.from_scenario(product_lib, text)
    cpu = oracle.OracleSim.from_scenario(text)
    assert_state_equal(gpu, cpu, f"{name} seed")
    for step in range(10):
        moved_gpu = gpu.run(10)
        moved_cpu = cpu.run(10)
        np.testing.assert_array_equal(moved_gpu, moved_cpu, err_msg=f"{name} moved counts")
        assert_state_equal(gpu, cpu, f"{name} tick {10 * (step + 1)}")
    gpu.verify()


@pytest.mark.parametrize("name", sorted(sc.EXTRA))
def test_extra_scenarios_free_run(product_lib, name):
    """Closed boundaries, 3x3 / 5x3 bodies, 21x21 and non-square fields, a field larger than the
    grid, linear regulation, every chunk width, non-default weights, ragged grid sizes."""
    text = sc.EXTRA[name]
    gpu = shim.Sim.from_scenario(product_lib, text)
    cpu = oracle.OracleSim.from_scenario(text)
    assert_state_equal(gpu, cpu, f"{name} seed")
    for step in range(6):
        np.testing.assert_array_equal(gpu.run(5), cpu.run(5), err_msg=f"{name} moved")
        assert_state_equal(gpu, cpu, f"{name} tick {5 * (step + 1)}")


@pytest.mark.parametrize("name", ["desk64", "closed-ped3", "k16", "linear-regulation", "ped5"])
def test_phase_by_phase_lockstep(product_lib, name):
    """Inspector path: after every phase the engine's temporaries equal the oracle's — decisions
    and f64 scores (k-2), enrollment table (k-2), vote winners (k-3), movement log, occupancy and
    centres (k-4), images (k-5) — with the GPU state overwritten from the CPU state each tick
    ("driven from the same field state")."""
    text = sc.DESK64 if name == "desk64" else sc.EXTRA[name]
    gpu = shim.Sim.from_scenario(product_lib, text)
    cpu = oracle.OracleSim.from_scenario(text)
    for tick in range(8):
        gpu.set_occupancy(cpu.occupancy())
        for k in range(3):
            gpu.set_image(k, cpu.image(k))
        gpu.set_centers(cpu.centers())
        gpu.tick = cpu.tick
        probe = cpu.clone()
        probe.step(until_phase=2)
        cap = gpu.step_capture()
        assert cap.phases_seen == 0b111110
        np.testing.assert_array_equal(cap.decisions, probe.decisions(), err_msg=f"tick {tick} decisions")
        np.testing.assert_array_equal(cap.enroll_ids, probe.enroll_ids(), err_msg=f"tick {tick} enrollment ids")
        np.testing.assert_array_equal(bits(cap.enroll_scores), bits(probe.enroll_scores()),
                                      err_msg=f"tick {tick} enrollment scores")
        full = cpu.clone()
        full.step(until_phase=4)
        np.testing.assert_array_equal(cap.winners, full.winners(), err_msg=f"tick {tick} winners")
        np.testing.assert_array_equal(cap.moved_from, full.moved_from(), err_msg=f"tick {tick} moved_from")
        np.testing.assert_array_equal(cap.moved_to, full.moved_to(), err_msg=f"tick {tick} moved_to")
        np.testing.assert_array_equal(cap.from_mask, full.from_mask(), err_msg=f"tick {tick} from_mask")
        np.testing.assert_array_equal(cap.to_mask, full.to_mask(), err_msg=f"tick {tick} to_mask")
        np.testing.assert_array_equal(cap.occupancy_k4.reshape(cpu.height, cpu.width), full.occupancy())
        np.testing.assert_array_equal(cap.centers_k4.reshape(-1, 2), full.centers())
        moved = cpu.step()
        assert cap.moved == moved
        assert_state_equal(gpu, cpu, f"{name} tick {tick + 1}")


def test_against_compiled_reference(product_lib, ref_lib):
    """The same comparison against the unmodified reference binary (oracle/_ref), both through
    the identical shim — the drop-in check: states_identical across implementations."""
    for text in (sc.DESK64, sc.EXTRA["closed-four"], sc.EXTRA["ped5"]):
        gpu = shim.Sim.from_scenario(product_lib, text)
        ref = shim.Sim.from_scenario(ref_lib, text, workers=2)
        for _ in range(4):
            np.testing.assert_array_equal(gpu.run(15), ref.run(15, mode="par"))
            assert gpu.digest() == ref.digest()
            np.testing.assert_array_equal(gpu.centers(), ref.centers())
            for k in range(3):
                np.testing.assert_array_equal(bits(gpu.image(k)), bits(ref.image(k)))


@pytest.mark.parametrize("knob,dense", [("0", "gather"), ("100000", "gather"), ("3", "gather"), ("3", "listwalk")])
@pytest.mark.parametrize("name", ["desk64", "k2", "k4", "k16", "field-5x9", "field-bigger-than-grid", "closed-four",
                                  "wide-ragged", "d0.1-eight-ped1", "d0.9-four-ped3", "field13-crowd"])
def test_both_k5_formulations(product_lib, monkeypatch, name, knob, dense):
    """The scatter path of k-5 chooses per tile by the number of movers in reach: an event-centric
    scatter (sparse tiles) or a dense kernel — the event-walk gather or the list walk.
    SFC_K5_EVENT_MAX forces every tile through one or the other (0: the gather alone, 100000: the
    scatter alone, 3: nearly every tile handed to the dense kernel); all bit-identical to the oracle."""
    monkeypatch.setenv("SFC_K5_PATH", "scatter")
    monkeypatch.setenv("SFC_K5_DENSE", dense)
    monkeypatch.setenv("SFC_K5_EVENT_MAX", knob)
    text = sc.DESK64 if name == "desk64" else sc.EXTRA.get(name) or dict(sc.acceptance3_scenarios())[name]
    gpu = shim.Sim.from_scenario(product_lib, text)
    cpu = oracle.OracleSim.from_scenario(text)
    for step in range(4):
        np.testing.assert_array_equal(gpu.run(8), cpu.run(8), err_msg=f"{name} moved")
        assert_state_equal(gpu, cpu, f"{name} knob {knob} tick {8 * (step + 1)}")


@pytest.mark.parametrize("path,knob", [("window", None), ("window", "100000"), ("window", "2"), ("scatter-list", None),
                                       ("listwalk", None), ("listwalk-list", None), ("pairs", None), ("pairs-list", None)])
@pytest.mark.parametrize("name", ["desk64", "k2", "k16", "field-5x9", "field21", "field-bigger-than-grid", "closed-four",
                                  "closed-ped3", "ped5", "wide-ragged", "sparse-periodic", "sparse-closed", "sparse-field15",
                                  "d0.9-four-ped3"])
def test_k5_active_tiles_and_window_kernel(product_lib, monkeypatch, name, path, knob):
    """k-4 lists the 32 x 8 tiles within field reach of a mover and k-5 visits only those; sparse
    crowds also switch to the window kernel (one warp per 8 x 4 su block, event-major scatter, exact
    replay).  Forced here on crowds of every density: the window kernel with its default hand-off
    to the dense gather, with every tile kept (knob 100000) or nearly every tile handed off (2), and
    the scatter kernel driven from the list, the list-walk kernel alone over every tile and over the
    listed tiles, the pair kernel (default for fields up to 9 su wide) over every tile and over the
    listed tiles.  All bit-identical to the oracle."""
    monkeypatch.setenv("SFC_K5_PATH", path.split("-")[0])
    if path.endswith("-list"):
        monkeypatch.setenv("SFC_K5_ACTIVE_LIST", "1")
    if knob is not None:
        monkeypatch.setenv("SFC_K5_EVENT_MAX", knob)
    text = sc.DESK64 if name == "desk64" else sc.EXTRA.get(name) or dict(sc.acceptance3_scenarios())[name]
    gpu = shim.Sim.from_scenario(product_lib, text)
    cpu = oracle.OracleSim.from_scenario(text)
    for step in range(4):
        np.testing.assert_array_equal(gpu.run(8), cpu.run(8), err_msg=f"{name} moved")
        assert_state_equal(gpu, cpu, f"{name} {path} knob {knob} tick {8 * (step + 1)}")


@pytest.mark.parametrize("red", ["0", "1"])
@pytest.mark.parametrize("name", ["desk64", "k2", "k4", "k16", "field-5x9", "closed-four", "wide-ragged", "sparse-periodic",
                                  "d0.9-eight-ped1", "d0.5-bi-ped3"])
def test_pair_kernel_image_update_variants(product_lib, monkeypatch, name, red):
    """The pair kernel adds (float)total to the image either as a plain read-modify-write or as a
    float reduction at the L2 (chosen when no image value can be subnormal — the reduction flushes
    them); both forced here, both bit-identical to the oracle."""
    monkeypatch.setenv("SFC_K5_PATH", "pairs")
    monkeypatch.setenv("SFC_K5_RED", red)
    text = sc.DESK64 if name == "desk64" else sc.EXTRA.get(name) or dict(sc.acceptance3_scenarios())[name]
    gpu = shim.Sim.from_scenario(product_lib, text)
    cpu = oracle.OracleSim.from_scenario(text)
    for step in range(4):
        np.testing.assert_array_equal(gpu.run(8), cpu.run(8), err_msg=f"{name} moved")
        assert_state_equal(gpu, cpu, f"{name} red {red} tick {8 * (step + 1)}")


def test_subnormal_image_values_stay_exact(product_lib):
    """Uploaded images holding subnormal / tiny values: sums can be subnormal, which a float
    reduction would flush — the engine must notice at upload and keep the exact path."""
    text = sc.variant(sc.DESK64, rebuild_interval=0)
    gpu = shim.Sim.from_scenario(product_lib, text)
    cpu = oracle.OracleSim.from_scenario(text)
    rng = np.random.default_rng(5)
    for k in range(3):
        img = cpu.image(k).copy()
        tiny = rng.random(img.shape) < 0.3
        img[tiny] = (rng.integers(1, 1 << 20, size=int(tiny.sum())).astype(np.uint32)).view(np.float32)  # subnormals
        cpu.image(k)[:] = img  # (a view of the oracle's memory)
        gpu.set_image(k, img)
    for step in range(3):
        np.testing.assert_array_equal(gpu.run(4), cpu.run(4))
        assert_state_equal(gpu, cpu, f"subnormal tick {4 * (step + 1)}")


@pytest.mark.parametrize("path", ["pairs", "scatter", "window", "field", "slabs", "bands"])
def test_negative_zero_image_entries_are_normalised_like_the_reference(product_lib, monkeypatch, path):
    """The reference's k-5 adds (float)total to EVERY (su, kind, sect) address once anybody moved
    (engine.cpp:468,524): a -0.0f entry — only reachable through the public mutable SimState — becomes
    +0.0f at the first moving tick, and stays -0.0f while nobody moves.  The device kernels skip
    untouched addresses, so a normalising pass follows the first moving tick: bit-identical images."""
    if path == "slabs":
        monkeypatch.setenv("SFC_SLABS", "2")
    elif path == "bands":
        monkeypatch.setenv("SFC_BANDS", "2")
    else:
        monkeypatch.setenv("SFC_K5_PATH", path)
    text = sc.variant(sc.DESK64, rebuild_interval=0, density=0.05, walk_period="3..3")
    gpu = shim.Sim.from_scenario(product_lib, text)
    cpu = oracle.OracleSim.from_scenario(text)
    rng = np.random.default_rng(11)
    for k in range(3):
        img = cpu.image(k).copy()
        zero = (img == 0.0) & (rng.random(img.shape) < 0.4)
        img[zero] = -0.0
        assert np.signbit(img[zero]).all()
        cpu.image(k)[:] = img
        gpu.set_image(k, img)
    for step in range(4):
        np.testing.assert_array_equal(gpu.run(2), cpu.run(2))
        assert_state_equal(gpu, cpu, f"negative zero, {path}, tick {2 * (step + 1)}")


def test_nan_scores_order_like_the_reference(product_lib):
    """NaN image values (only reachable through the public mutable SimState) give NaN scores, which the
    reference's vote orders by slot position: the first registrant seeds the best, a later NaN never
    beats it, a seeded NaN is never beaten (engine.cpp:365-386).  The vote here is the same scan, so
    decisions, winners and positions agree; the images agree wherever they are numbers (a NaN's payload
    is not portable between x86 and the GPU's adders)."""
    text = sc.variant(sc.DESK64, rebuild_interval=0, density=0.6)
    gpu = shim.Sim.from_scenario(product_lib, text)
    cpu = oracle.OracleSim.from_scenario(text)
    rng = np.random.default_rng(12)
    for k in range(3):
        img = cpu.image(k).copy()
        img[rng.random(img.shape) < 0.02] = np.nan
        cpu.image(k)[:] = img
        gpu.set_image(k, img)
    for step in range(5):
        np.testing.assert_array_equal(gpu.run(3), cpu.run(3), err_msg="moved")
        np.testing.assert_array_equal(gpu.centers(), cpu.centers(), err_msg=f"tick {gpu.tick} centres")
        np.testing.assert_array_equal(gpu.occupancy(), cpu.occupancy(), err_msg=f"tick {gpu.tick} occupancy")
        for k in range(3):
            a, b = gpu.image(k), cpu.image(k)
            np.testing.assert_array_equal(np.isnan(a), np.isnan(b))
            np.testing.assert_array_equal(bits(np.where(np.isnan(a), 0.0, a).astype(np.float32)),
                                          bits(np.where(np.isnan(b), 0.0, b).astype(np.float32)))


@pytest.mark.parametrize("name", ["desk64", "field21", "d0.9-eight-ped1", "closed-four"])
def test_rebuild_with_more_centres_than_its_sorted_list_holds(product_lib, monkeypatch, name):
    """The rebuild sorts the centres of a tile's region by id in shared memory; when a region holds more
    than the list does (large fields in dense crowds), it takes them in rounds of ascending id ranges —
    the per-address order is ascending id either way.  Forced with a 32-entry list; bit-identical."""
    monkeypatch.setenv("SFC_REBUILD_CAP", "32")
    text = sc.variant(sc.DESK64 if name == "desk64" else sc.EXTRA.get(name) or dict(sc.acceptance3_scenarios())[name], rebuild_interval=3)
    gpu = shim.Sim.from_scenario(product_lib, text)  # (seeding rasterises through the same kernel)
    cpu = oracle.OracleSim.from_scenario(text)
    assert_state_equal(gpu, cpu, f"{name} seed")
    for step in range(3):
        np.testing.assert_array_equal(gpu.run(4), cpu.run(4))
        assert_state_equal(gpu, cpu, f"{name} tick {4 * (step + 1)}")


def test_default_path_field13(product_lib):
    """13 x 13 fields in a crowd, no knobs: scatter kernel, crowded tiles handed to the list walk."""
    text = sc.EXTRA["field13-crowd"]
    gpu = shim.Sim.from_scenario(product_lib, text)
    cpu = oracle.OracleSim.from_scenario(text)
    for step in range(3):
        np.testing.assert_array_equal(gpu.run(5), cpu.run(5))
        assert_state_equal(gpu, cpu, f"field13 tick {5 * (step + 1)}")


@pytest.mark.parametrize("name,ticks,list_cap", [("field35", 8, None), ("field41-crowd", 4, None), ("field35", 6, "16")])
def test_large_field_gather(product_lib, monkeypatch, name, ticks, list_cap):
    """Fields beyond 15 x 15 (BASELINE configs 3 and 5 use 35 x 35 and 77 x 77) take the event-walk
    gather on 32 x 16 tiles whose field region is staged in column chunks: one sorted event list per
    tile when the events fit, re-staging per walk when they do not (forced with a 16-event list).
    Bit-identical to the oracle."""
    monkeypatch.setenv("SFC_K5_PATH", "scatter")  # (the default for these fields is the field kernel, below)
    if list_cap:
        monkeypatch.setenv("SFC_K5_LIST_CAP", list_cap)
    text = sc.EXTRA[name]
    gpu = shim.Sim.from_scenario(product_lib, text)
    cpu = oracle.OracleSim.from_scenario(text)
    for step in range(2):
        np.testing.assert_array_equal(gpu.run(ticks // 2), cpu.run(ticks // 2), err_msg=f"{name} moved")
        assert_state_equal(gpu, cpu, f"{name} tick {(step + 1) * (ticks // 2)}")


FIELD_VARIANTS = [  # (kinds per walk, warps per CTA, lazy partials, list capacity); None = the engine's choice
    (None, None, None, None), ("3", "4", "0", None), ("3", "4", "1", None), ("1", "8", "0", None), ("1", "8", "1", None),
    ("1", "4", "1", "48"), ("3", "4", "0", "48"), ("1", "16", "0", None),
]


@pytest.mark.parametrize("nk,warps,lazy,cap", FIELD_VARIANTS)
@pytest.mark.parametrize("name", ["desk64", "k2", "k4", "k16", "field-5x9", "field21", "field-bigger-than-grid", "closed-four",
                                  "closed-ped3", "field35", "field41-crowd", "field13-crowd", "wide-ragged", "sparse-closed",
                                  "weights", "d0.9-eight-ped1"])
def test_field_kernel(product_lib, monkeypatch, name, nk, warps, lazy, cap):
    """The large-field kernel (default beyond 15 x 15: BASELINE configs 3 and 5) forced on fields of
    every size and crowds of every density, in each of its shapes: three kinds per walk or one, four,
    eight or sixteen warps per CTA (tiles of 32 x 2 / 4 / 8 su), partials cleared per block or created
    lazily, and with 48-event lists so the region streams through many column chunks.  All
    bit-identical to the oracle."""
    monkeypatch.setenv("SFC_K5_PATH", "field")
    for knob, value in (("SFC_K5_FIELD_NK", nk), ("SFC_K5_FIELD_WARPS", warps), ("SFC_K5_FIELD_LAZY", lazy), ("SFC_K5_LIST_CAP", cap)):
        if value is not None:
            monkeypatch.setenv(knob, value)
    if name == "k16" and warps == "16":
        pytest.skip("sixteen warps of sixteen-slot partials exceed shared memory")
    monkeypatch.setenv("SFC_K5_STRICT", "1")  # a forced path that cannot be honoured is an error, not a silent fallback
    text = sc.DESK64 if name == "desk64" else sc.EXTRA.get(name) or dict(sc.acceptance3_scenarios())[name]
    gpu = shim.Sim.from_scenario(product_lib, text)
    cpu = oracle.OracleSim.from_scenario(text)
    ticks = 4 if "field4" in name or "field35" in name else 8
    for step in range(3):
        np.testing.assert_array_equal(gpu.run(ticks), cpu.run(ticks), err_msg=f"{name} moved")
        assert_state_equal(gpu, cpu, f"{name} nk {nk} warps {warps} lazy {lazy} cap {cap} tick {ticks * (step + 1)}")


@pytest.mark.parametrize("name", ["desk64", "closed-ped3", "d0.9-eight-ped1", "linear-regulation", "sparse-periodic", "wide-ragged"])
def test_position_ordered_pedestrian_kernels(product_lib, monkeypatch, name):
    """k-2 ... k-4 visiting the pedestrians in row-major order of their centres (PedArrays::order, the engine's
    choice on grids from 2^28 su; forced here) instead of id order: every tie-break is on the id
    (engine.cpp:375-378), so nothing may change.  120 ticks cross two re-ordering passes and two rebuilds;
    multi-cell pedestrians make sure only centres are listed."""
    monkeypatch.setenv("SFC_PED_ORDER", "1")
    text = sc.DESK64 if name == "desk64" else sc.EXTRA.get(name) or dict(sc.acceptance3_scenarios())[name]
    gpu = shim.Sim.from_scenario(product_lib, text)
    cpu = oracle.OracleSim.from_scenario(text)
    for step in range(4):
        np.testing.assert_array_equal(gpu.run(30), cpu.run(30), err_msg=f"{name} moved")
        assert_state_equal(gpu, cpu, f"{name} position order tick {30 * (step + 1)}")


@pytest.mark.parametrize("path", ["window", "scatter-list", "listwalk-list", "pairs-list"])
@pytest.mark.parametrize("name", ["sparse-periodic", "sparse-closed", "closed-ped3"])
def test_rebuild_skips_only_untouched_tiles(product_lib, monkeypatch, name, path):
    """With the active-tile stamps on, a rebuild leaves alone the tiles no mover has reached since the previous
    rebuild (their images are still that rebuild's fresh ones, bit for bit).  Rebuilds every 7 ticks, also
    across the stamp period (erased stamps: that rebuild must look at every tile) and across separate runs;
    oracle-identical after every rebuild, and identical to the same engine with skipping off."""
    monkeypatch.setenv("SFC_K5_PATH", path.split("-")[0])
    if path.endswith("-list"):
        monkeypatch.setenv("SFC_K5_ACTIVE_LIST", "1")
    text = sc.variant(sc.EXTRA[name], rebuild_interval=7)
    gpu = shim.Sim.from_scenario(product_lib, text)
    cpu = oracle.OracleSim.from_scenario(text)
    for start in (0, 65535 - 10):
        gpu.tick = cpu.tick = start
        for ticks in (7, 14, 3, 4, 8):
            np.testing.assert_array_equal(gpu.run(ticks), cpu.run(ticks))
            assert_state_equal(gpu, cpu, f"{name} {path} tick {gpu.tick}")


@pytest.mark.parametrize("path", ["window", "scatter-list", "listwalk-list", "pairs-list"])
def test_tile_stamps_survive_the_epoch_period(product_lib, monkeypatch, path):
    """The active-tile stamps carry the tick modulo 65535; the engine erases them once per period so
    a stamp from exactly one period ago cannot pass for the current tick.  Run across the boundary
    (and once more across it in a second run) with every list-driven k-5 path."""
    monkeypatch.setenv("SFC_K5_PATH", path.split("-")[0])
    if path.endswith("-list"):
        monkeypatch.setenv("SFC_K5_ACTIVE_LIST", "1")
    text = sc.variant(sc.EXTRA["sparse-periodic"], rebuild_interval=0)
    gpu = shim.Sim.from_scenario(product_lib, text)
    cpu = oracle.OracleSim.from_scenario(text)
    for start in (65531, 2 * 65535 - 3):
        gpu.tick = cpu.tick = start
        for _ in range(3):
            np.testing.assert_array_equal(gpu.run(3), cpu.run(3))
            assert_state_equal(gpu, cpu, f"{path} tick {gpu.tick}")
