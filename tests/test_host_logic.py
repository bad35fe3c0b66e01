"""CPU-side checks of the product: the C ABI exports what include/socfield_cuda.h declares, the
host mirror builds the same tables as the oracle, the scenario parser keeps the reference's
grammar and error behaviour, and the Python module keeps the reference's surface.  No GPU
compute is invoked here (the library loads and is introspected only)."""
import ctypes
import os
import re

import numpy as np
import pytest

from oracle import oracle
from paper_1803_04782_b200 import library_path
from paper_1803_04782_b200 import socfield as sf

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_c_abi_exports_every_declared_symbol():
    header = open(os.path.join(ROOT, "include", "socfield_cuda.h")).read()
    declared = set(re.findall(r"\b(sfc_[a-z_]+)\s*\(", header))
    assert {"sfc_create", "sfc_upload", "sfc_run", "sfc_phase", "sfc_download", "sfc_destroy",
            "sfc_download_temporaries", "sfc_rasterize_dynamic", "sfc_rasterize_static", "sfc_decide",
            "sfc_last_error"} <= declared
    lib = ctypes.CDLL(library_path("libsocfield_cuda.so"))
    for name in sorted(declared):
        assert hasattr(lib, name), f"{name} declared in socfield_cuda.h but not exported"
    lib.sfc_abi_version.restype = ctypes.c_int
    assert lib.sfc_abi_version() == 1
    lib.sfc_device_count.restype = ctypes.c_int
    assert lib.sfc_device_count() >= 0


def test_no_cpu_fallback_without_device():
    if sf.device_count() > 0:
        pytest.skip("a CUDA device is present")
    cfg = sf.parse_scenario("grid = 16x16\ndensity = 0.2\n")
    with pytest.raises(RuntimeError, match="no CUDA device"):
        sf.Engine(cfg)
    with pytest.raises(RuntimeError, match="no CUDA device"):
        sf.seed_population(cfg)  # the initial images are rasterised on the device


def test_python_surface_matches_reference_module():
    """Names bound by the reference's pybind module (bindings/module.cpp:62-346)."""
    for name in ["GridGeometry", "wrap", "footprint_cells", "sect_index", "sect_distance", "FieldSpec", "strength_at",
                 "support", "WritePlan", "build_write_plan", "fanout_brute_force", "one_step_sum", "multi_step_sum",
                 "chunk_count", "sort8_desc", "ScenarioConfig", "parse_scenario", "parse_scenario_file",
                 "serialize_scenario", "validate_scenario", "planned_population", "scale_fields", "SimState",
                 "seed_population", "states_identical", "TickMetrics", "Engine", "ParseError", "ConfigError",
                 "SeedingError", "IntegrityError", "MemoryPlan", "memory_plan"]:
        assert hasattr(sf, name), name
    for method in ["tick", "run", "verify_state", "plan_fanout"]:
        assert hasattr(sf.Engine, method)
    for method in ["occupancy", "image", "centers", "copy"]:
        assert hasattr(sf.SimState, method)


def test_reference_smoke_cases_host_side():
    """The host-only cases of the reference's tests/python/test_smoke.py."""
    grid = sf.GridGeometry(100, 100)
    assert sf.wrap(grid, 100, -1) == (0, 99)
    assert sf.wrap(sf.GridGeometry(10, 10, "closed"), 10, 3) is None
    assert sf.sect_index(1, 0) == 0 and sf.sect_index(1, 1) == 1 and sf.sect_index(3, 2) == 1
    assert sf.sect_index(0, 0) is None
    rng = np.random.default_rng(7)
    terms = rng.uniform(-5, 5, size=481).tolist()
    one = sf.one_step_sum(terms)
    for k in (2, 4, 8, 16):
        assert sf.multi_step_sum(terms, k) == pytest.approx(one, rel=1e-9, abs=1e-9)
    assert sf.chunk_count(48, 8) == 6
    with pytest.raises(Exception):
        sf.multi_step_sum(terms, 3)
    field = sf.FieldSpec("recurrent-repulsive", (7, 7), gain=1.0, decay=-0.5)
    plan = sf.build_write_plan(field)
    assert plan.fanout == sf.fanout_brute_force(field) == 7
    assert sum(len(plan.contributors(s)) for s in range(8)) == len(sf.support(field)) == 48
    assert sf.sort8_desc([0.0] * 8) == list(range(8))
    assert sf.sort8_desc([1, 2, 3, 4, 5, 6, 7, 8]) == [7, 6, 5, 4, 3, 2, 1, 0]
    cfg = sf.parse_scenario("grid = 32x32\ndensity = 0.5\nseed = 9\n")
    assert sf.parse_scenario(sf.serialize_scenario(cfg)).density == 0.5
    assert sf.planned_population(cfg) == 512
    with pytest.raises(Exception, match="density"):
        sf.parse_scenario("grid = 10x10\ndensity = 1.5\n")


def test_host_sort8_and_multi_step_sum_equal_oracle():
    L = oracle.lib()
    rng = np.random.default_rng(3)
    for trial in range(500):
        s = rng.uniform(-1, 1, 8) if trial % 2 else rng.integers(0, 3, 8).astype(float)
        a = (ctypes.c_double * 8)(*s)
        o = (ctypes.c_int32 * 8)()
        L.so_sort8_desc(a, o)
        assert sf.sort8_desc(list(s)) == list(o)
    terms = rng.uniform(-3, 3, 1000)
    for k in (2, 4, 8, 16):
        assert sf.multi_step_sum(terms.tolist(), k) == L.so_multi_step_sum(terms.ctypes.data, terms.size, k)


@pytest.mark.parametrize("geom", [(7, 7), (5, 9), (21, 21), (1, 1), (3, 1)])
@pytest.mark.parametrize("gain,decay", [(1.0, -0.5), (1.3, -0.37)])
def test_write_plans_and_device_tables_equal_oracle(geom, gain, decay):
    """build_write_plan (API) and the flat contributor table uploaded to the device
    (socfield_cuda.h sfc_kind_table) against the oracle's plans / gather lists, bit for bit."""
    cfg = oracle.make_config(16, 16, templates=[(geom[0], geom[1], gain, decay)] * 3)
    cpu = oracle.OracleSim.from_arrays(cfg, [])
    hw, hh = geom[0] // 2, geom[1] // 2
    for kind, name in enumerate(("dir-attractive", "dir-repulsive", "recurrent-repulsive")):
        for orient in range(8):
            plan = sf.build_write_plan(sf.FieldSpec(name, geom, gain, decay, orient))
            for sect in range(8):
                dxdy, mag = cpu.plan_entries(kind, orient, sect)
                got = plan.contributors(sect)
                assert [tuple(c[0]) for c in got] == [tuple(d) for d in dxdy.tolist()]
                assert np.array_equal(np.array([c[1] for c in got], np.float64).view(np.uint64), mag.view(np.uint64))
        tmag, tinfo = sf._kind_table(sf.FieldSpec(name, geom, gain, decay))
        seen = 0
        for sect in range(8):
            dxdy, mag, mask = cpu.gather_entries(kind, sect)
            for j, (d, m, ms) in enumerate(zip(dxdy, mag, mask)):
                info = int(tinfo[d[1] + hh, d[0] + hw])
                assert (info & 7, (info >> 3) & 0xFF, info >> 11) == (sect, int(ms), j)
                assert tmag[d[1] + hh, d[0] + hw] == m
                seen += 1
        assert seen == int(((tinfo >> 3) & 0xFF != 0).sum())


def test_scenario_grammar_and_errors():
    """Reference scenario.cpp:172-268: comments, unknown / duplicate keys with line numbers,
    constraint errors naming the field; serialize/parse round trip (:278-307)."""
    cfg = sf.parse_scenario("# c\n grid = 12x8   # trailing\n\nboundary = closed\nwalk_period = 2..5\nseed = 18446744073709551615\n")
    assert (cfg.grid.width, cfg.grid.height, cfg.grid.boundary) == (12, 8, "closed")
    assert (cfg.walk_period_min, cfg.walk_period_max, cfg.seed) == (2, 5, 2**64 - 1)
    text = sf.serialize_scenario(cfg)
    assert sf.serialize_scenario(sf.parse_scenario(text)) == text
    with pytest.raises(sf.ParseError, match=r"line 2: unknown key 'colour'"):
        sf.parse_scenario("grid = 8x8\ncolour = red\n")
    with pytest.raises(sf.ParseError, match=r"line 3: duplicate key 'grid' \(first on line 1\)"):
        sf.parse_scenario("grid = 8x8\ndensity = 0.5\ngrid = 9x9\n")
    with pytest.raises(sf.ParseError, match="expected 'key = value'"):
        sf.parse_scenario("grid 8x8\n")
    with pytest.raises(sf.ParseError, match="trailing characters"):
        sf.parse_scenario("ticks = 12abc\n")
    with pytest.raises(sf.ParseError, match="expected WIDTHxHEIGHT"):
        sf.parse_scenario("grid = 88\n")
    for text, field in [("chunk_k = 3\n", "chunk_k"), ("field_geometry = 6x7\n", "field_geometry"),
                        ("density = 0\n", "density"), ("walk_period = 3..2\n", "walk_period"),
                        ("boundary = open\n", "boundary"), ("grid = 4x4\npedestrian_geometry = 5x5\n", "pedestrian_geometry"),
                        ("grid = 4x4\ndensity = 0.1\ndirections = eight\n", "density")]:
        with pytest.raises(sf.ConfigError, match=field):
            sf.parse_scenario(text)
    assert sf.scale_fields(cfg, 3) == (21, 21)
    with pytest.raises(sf.ConfigError):
        sf.scale_fields(cfg, 2)
    # exact population literals of the big bench configs
    c3 = sf.parse_scenario("grid = 8192x8192\ndensity = 0.00298023223876953125\nfield_geometry = 35x35\n")
    c4 = sf.parse_scenario("grid = 32768x32768\ndensity = 0.000931322574615478515625\n")
    assert sf.planned_population(c3) == 200000 and sf.planned_population(c4) == 1000000


def test_strength_law_equals_oracle():
    import ctypes as C

    L = oracle.lib()
    for kind_i, kind in [(2, "dir-attractive"), (3, "dir-repulsive"), (4, "recurrent-repulsive"), (0, "omni-attractive"),
                         (1, "omni-repulsive")]:
        f = sf.FieldSpec(kind, (9, 7), 1.7, -0.3, 5)
        of = oracle.SoField(9, 7, 1.7, -0.3)
        grid = sf.GridGeometry(64, 64)
        for dx in range(-5, 6):
            for dy in range(-4, 5):
                sx, sy = C.c_double(), C.c_double()
                L.so_strength_at_offset(kind_i, C.byref(of), 5, dx, dy, C.byref(sx), C.byref(sy))
                assert sf.strength_at(f, (20, 20), (20 + dx, 20 + dy), grid) == (sx.value, sy.value)


def test_memory_plan_numbers_and_errors():
    """memory_plan (reference bench.cpp:14-24): paper section 3.2's one-step cache arithmetic — the
    reference's own cases (test_bench_cli.cpp:41-67, tests/python/test_smoke.py:9-15)."""
    grid = sf.GridGeometry(1000, 1000)
    for fanout, m_recur, gib in [(6, 192, 0.7), (61, 1952, 7.3), (164, 5248, 19.6), (328, 10496, 39.1), (535, 17120, 63.8),
                                 (808, 25856, 96.3)]:
        plan = sf.memory_plan(fanout, grid)
        assert plan.sf == fanout and plan.m_recur_bytes == m_recur and plan.m_total_bytes == 4 * m_recur
        assert plan.grid_bytes == plan.m_total_bytes * 1_000_000
        assert abs(plan.gib_display - gib) <= 0.05
    zero = sf.memory_plan(0, grid)
    assert (zero.m_recur_bytes, zero.m_total_bytes, zero.grid_bytes, zero.gib) == (0, 0, 0, 0.0)
    with pytest.raises(sf.ConfigError):
        sf.memory_plan(-1, sf.GridGeometry(10, 10))
    # BASELINE config 3 (35 x 35 fields: fan-out 179 on 8192^2): the one-step cache would need 1432 GiB
    assert round(sf.memory_plan(179, sf.GridGeometry(8192, 8192)).gib) == 1432
