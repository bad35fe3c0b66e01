"""ctypes front end for the plain-C oracle (oracle/socfield_oracle.c).

TEST INFRASTRUCTURE — the CPU restatement of the reference's per-tick path.  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / reference arm may import this.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "build", "libsocfield_oracle.so")


class SoField(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("gain", C.c_double), ("decay", C.c_double)]


class SoConfig(C.Structure):
    _fields_ = [
        ("width", C.c_int32), ("height", C.c_int32), ("closed", C.c_int32),
        ("chunk_k", C.c_int32),
        ("weight_static", C.c_double), ("weight_dir_attractive", C.c_double),
        ("weight_dir_repulsive", C.c_double), ("weight_recurrent", C.c_double), ("goal_bias", C.c_double),
        ("regulation", C.c_int32), ("density_radius", C.c_int32),
        ("rebuild_interval", C.c_int64), ("rebuild_tolerance", C.c_double),
        ("fault_invert_vote_tiebreak", C.c_int32),
        ("templates", SoField * 3),
    ]


class SoSeedSpec(C.Structure):
    _fields_ = [
        ("density", C.c_double), ("n_goal_sects", C.c_int32), ("goal_sects", C.c_int32 * 8),
        ("ped_width", C.c_int32), ("ped_height", C.c_int32),
        ("walk_period_min", C.c_int32), ("walk_period_max", C.c_int32), ("seed", C.c_uint64),
    ]


class SoAnchor(C.Structure):
    _fields_ = [("kind", C.c_int32), ("width", C.c_int32), ("height", C.c_int32), ("gain", C.c_double),
                ("decay", C.c_double), ("x", C.c_int32), ("y", C.c_int32)]


DIRECTION_SECTS = {"uni": [0], "bi": [0, 4], "four": [0, 2, 4, 6], "eight": list(range(8))}

# ScenarioConfig defaults, reference scenario.hpp:21-47
SCENARIO_DEFAULTS = dict(
    grid=(100, 100), boundary="periodic", density=0.5, directions="eight", field_geometry=(7, 7),
    pedestrian_geometry=(1, 1), walk_period=(1, 1), chunk_k=8, ticks=100, repeats=3, seed=42,
    field_gain=1.0, field_decay=-0.5, weight_static=1.0, weight_dir_attractive=1.0,
    weight_dir_repulsive=1.0, weight_recurrent=1.0, goal_bias=1.0, regulation="identity",
    density_radius=3, rebuild_interval=50,
)


def parse_scenario_text(text: str) -> dict:
    """Minimal reader of the reference's `key = value` scenario format (scenario.cpp:172-268),
    for feeding the flat-C oracle; validation lives in the product's parse_scenario."""
    cfg = dict(SCENARIO_DEFAULTS)
    for raw in text.splitlines():
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        key, value = [t.strip() for t in line.split("=", 1)]
        if key in ("grid", "field_geometry", "pedestrian_geometry"):
            w, h = value.split("x")
            cfg[key] = (int(w), int(h))
        elif key == "walk_period":
            lo, _, hi = value.partition("..")
            cfg[key] = (int(lo), int(hi or lo))
        elif key in ("boundary", "directions", "regulation"):
            cfg[key] = value
        elif key in ("density", "field_gain", "field_decay", "weight_static", "weight_dir_attractive",
                     "weight_dir_repulsive", "weight_recurrent", "goal_bias"):
            cfg[key] = float(value)
        elif key in ("chunk_k", "ticks", "repeats", "seed", "density_radius", "rebuild_interval", "version"):
            cfg[key] = int(value)
        else:
            raise ValueError(f"unknown key {key!r}")
    return cfg


def make_config(width, height, *, closed=False, chunk_k=8, weight_static=1.0, weight_dir_attractive=1.0,
                weight_dir_repulsive=1.0, weight_recurrent=1.0, goal_bias=1.0, regulation=0,
                density_radius=3, rebuild_interval=0, rebuild_tolerance=1e-4, fault_invert_vote_tiebreak=0,
                templates=None) -> SoConfig:
    templates = templates or [(7, 7, 1.0, -0.5)] * 3
    return SoConfig(width, height, int(closed), chunk_k, weight_static, weight_dir_attractive,
                    weight_dir_repulsive, weight_recurrent, goal_bias, regulation, density_radius,
                    rebuild_interval, rebuild_tolerance, fault_invert_vote_tiebreak,
                    (SoField * 3)(*[SoField(*t) for t in templates]))


def config_from_scenario(sc: dict) -> tuple[SoConfig, SoSeedSpec]:
    fg = sc["field_geometry"]
    cfg = make_config(sc["grid"][0], sc["grid"][1], closed=sc["boundary"] == "closed", chunk_k=sc["chunk_k"],
                      weight_static=sc["weight_static"], weight_dir_attractive=sc["weight_dir_attractive"],
                      weight_dir_repulsive=sc["weight_dir_repulsive"], weight_recurrent=sc["weight_recurrent"],
                      goal_bias=sc["goal_bias"], regulation=0 if sc["regulation"] == "identity" else 1,
                      density_radius=sc["density_radius"], rebuild_interval=sc["rebuild_interval"],
                      templates=[(fg[0], fg[1], sc["field_gain"], sc["field_decay"])] * 3)
    sects = DIRECTION_SECTS[sc["directions"]]
    spec = SoSeedSpec(sc["density"], len(sects), (C.c_int32 * 8)(*(sects + [0] * (8 - len(sects)))),
                      sc["pedestrian_geometry"][0], sc["pedestrian_geometry"][1], sc["walk_period"][0],
                      sc["walk_period"][1], sc["seed"])
    return cfg, spec


def build(force: bool = False) -> str:
    src = os.path.join(HERE, "socfield_oracle.c")
    hdr = os.path.join(HERE, "socfield_oracle.h")
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(src), os.path.getmtime(hdr)):
        subprocess.check_call(["make", "-s", "-C", HERE, "oracle"])
    return LIB


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    L = C.CDLL(build())
    vp, i32, i64, dbl = C.c_void_p, C.c_int32, C.c_int64, C.c_double
    sig = {
        "so_last_error": (C.c_char_p, [vp]), "so_error_phase": (C.c_int, [vp]),
        "so_create": (vp, [C.POINTER(SoConfig), i64, vp, vp, vp, vp, vp, vp, vp, C.c_char_p, C.c_size_t]),
        "so_seed": (vp, [C.POINTER(SoConfig), C.POINTER(SoSeedSpec), C.c_char_p, C.c_size_t]),
        "so_clone": (vp, [vp]), "so_free": (None, [vp]),
        "so_population": (i64, [vp]), "so_tick_count": (i64, [vp]), "so_set_tick": (None, [vp, i64]),
        "so_planned_population": (i64, [C.POINTER(SoConfig), C.POINTER(SoSeedSpec)]),
        "so_tick": (C.c_int, [vp, C.c_int, C.POINTER(i64)]),
        "so_run": (C.c_int, [vp, i64, vp]),
        "so_verify": (C.c_int, [vp]),
        "so_decide": (C.c_int, [vp, i64, C.POINTER(i32), C.POINTER(dbl)]),
        "so_rebuild_images": (None, [vp, vp]),
        "so_set_static_fields": (C.c_int, [vp, i64, C.POINTER(SoAnchor)]),
        "so_digest": (C.c_uint64, [vp]), "so_set_threads": (None, [C.c_int]),
        "so_occupancy": (C.POINTER(i32), [vp]), "so_image": (C.POINTER(C.c_float), [vp, C.c_int]),
        "so_centers_x": (C.POINTER(i32), [vp]), "so_centers_y": (C.POINTER(i32), [vp]),
        "so_ped_attr": (C.POINTER(i32), [vp, C.c_int]),
        "so_decisions": (C.POINTER(i32), [vp]), "so_decision_scores": (C.POINTER(dbl), [vp]),
        "so_enroll_ids": (C.POINTER(i32), [vp]), "so_enroll_scores": (C.POINTER(dbl), [vp]),
        "so_winners": (C.POINTER(i32), [vp]), "so_moved_from": (C.POINTER(i32), [vp]),
        "so_moved_to": (C.POINTER(i32), [vp]),
        "so_from_mask": (C.POINTER(C.c_uint8), [vp, C.c_int]), "so_to_mask": (C.POINTER(C.c_uint8), [vp, C.c_int]),
        "so_sect_index": (C.c_int, [dbl, dbl]), "so_sect_distance": (C.c_int, [C.c_int, C.c_int]),
        "so_strength_at_offset": (None, [C.c_int, C.POINTER(SoField), C.c_int, C.c_int, C.c_int,
                                         C.POINTER(dbl), C.POINTER(dbl)]),
        "so_sort8_desc": (None, [C.POINTER(dbl), C.POINTER(i32)]),
        "so_multi_step_sum": (dbl, [vp, i64, C.c_int]), "so_one_step_sum": (dbl, [vp, i64]),
        "so_local_density": (dbl, [vp, C.c_int, C.c_int, C.c_int]),
        "so_plan_entries": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, vp, vp, C.c_int]),
        "so_gather_entries": (C.c_int, [vp, C.c_int, C.c_int, vp, vp, vp, C.c_int]),
        "so_rng_check": (None, [C.c_uint64, C.c_int, C.c_int, C.c_int, vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype, fn.argtypes = res, args
    _lib = L
    return L


class OracleError(RuntimeError):
    def __init__(self, message, phase=0):
        super().__init__(message)
        self.phase = phase


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class OracleSim:
    """Flat-array CPU oracle for one (engine, state) pair."""

    def __init__(self, handle, cfg: SoConfig):
        self.L = lib()
        self.h = C.c_void_p(handle)
        self.cfg = cfg
        self.width, self.height, self.closed = cfg.width, cfg.height, bool(cfg.closed)
        self.cells = self.width * self.height

    @classmethod
    def from_arrays(cls, cfg: SoConfig, peds) -> "OracleSim":
        rows = []
        for p in peds:
            if isinstance(p, dict):
                rows.append((p["x"], p["y"], p.get("goal", 0), p.get("fw", 1), p.get("fh", 1),
                             p.get("period", 1), p.get("phase", 0)))
            else:
                p = tuple(p)
                rows.append(p + (0, 1, 1, 1, 0)[len(p) - 2:] if len(p) < 7 else p)
        n = len(rows)
        arr = np.array(rows, np.int32).reshape(n, 7) if n else np.zeros((0, 7), np.int32)
        cx, cy, goal, fw, fh, period, phase = [np.ascontiguousarray(arr[:, i]) for i in range(7)]
        err = C.create_string_buffer(256)
        h = lib().so_create(C.byref(cfg), n, _p(cx), _p(cy), _p(fw), _p(fh), _p(period), _p(phase), _p(goal),
                            err, len(err))
        if not h:
            raise OracleError(err.value.decode())
        return cls(h, cfg)

    @classmethod
    def from_scenario(cls, text: str) -> "OracleSim":
        cfg, spec = config_from_scenario(parse_scenario_text(text))
        err = C.create_string_buffer(256)
        h = lib().so_seed(C.byref(cfg), C.byref(spec), err, len(err))
        if not h:
            raise OracleError(err.value.decode())
        return cls(h, cfg)

    def clone(self) -> "OracleSim":
        return OracleSim(self.L.so_clone(self.h), self.cfg)

    def close(self):
        if self.h:
            self.L.so_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def population(self) -> int:
        return self.L.so_population(self.h)

    @property
    def tick(self) -> int:
        return self.L.so_tick_count(self.h)

    @tick.setter
    def tick(self, v: int):
        self.L.so_set_tick(self.h, v)

    def _raise(self):
        raise OracleError(self.L.so_last_error(self.h).decode(), self.L.so_error_phase(self.h))

    def step(self, until_phase: int = 0) -> int:
        moved = C.c_int64()
        if self.L.so_tick(self.h, until_phase, C.byref(moved)):
            self._raise()
        return moved.value

    def run(self, ticks: int) -> np.ndarray:
        moved = np.zeros(max(ticks, 0), np.int64)
        if self.L.so_run(self.h, ticks, _p(moved)):
            self._raise()
        return moved

    def verify(self):
        if self.L.so_verify(self.h):
            self._raise()

    def decide(self, ped: int):
        d, s = C.c_int32(), C.c_double()
        self.L.so_decide(self.h, ped, C.byref(d), C.byref(s))
        return d.value, s.value

    def rebuild_images(self) -> np.ndarray:
        out = np.zeros((3, self.height, self.width, 8), np.float32)
        self.L.so_rebuild_images(self.h, _p(out))
        return out

    def set_static_fields(self, anchors):
        anchors = list(anchors)
        arr = (SoAnchor * max(1, len(anchors)))(*[SoAnchor(*a) for a in anchors])
        self.L.so_set_static_fields(self.h, len(anchors), arr)

    def digest(self) -> int:
        return int(self.L.so_digest(self.h))

    @staticmethod
    def set_threads(n: int) -> None:
        """k-5 over n threads (static su partition, like the reference's parallel_for); results do not depend on n."""
        lib().so_set_threads(int(n))

    # views (numpy arrays aliasing the oracle's memory)
    def _view(self, ptr, shape, dtype):
        n = int(np.prod(shape))
        if n == 0:
            return np.zeros(shape, dtype)
        return np.ctypeslib.as_array(ptr, shape=(n,)).view(dtype).reshape(shape)

    def occupancy(self):
        return self._view(self.L.so_occupancy(self.h), (self.height, self.width), np.int32)

    def image(self, which: int):
        return self._view(self.L.so_image(self.h, which), (self.height, self.width, 8), np.float32)

    def images(self):
        return np.stack([self.image(k) for k in range(3)])

    def centers(self):
        p = self.population
        return np.stack([self._view(self.L.so_centers_x(self.h), (p,), np.int32),
                         self._view(self.L.so_centers_y(self.h), (p,), np.int32)], axis=1)

    def set_centers(self, xy):
        p = self.population
        self._view(self.L.so_centers_x(self.h), (p,), np.int32)[:] = xy[:, 0]
        self._view(self.L.so_centers_y(self.h), (p,), np.int32)[:] = xy[:, 1]

    def ped_attrs(self):
        p = self.population
        names = ("period", "phase", "goal", "fw", "fh")
        return {k: self._view(self.L.so_ped_attr(self.h, i), (p,), np.int32).copy() for i, k in enumerate(names)}

    def decisions(self):
        return self._view(self.L.so_decisions(self.h), (self.population,), np.int32).copy()

    def decision_scores(self):
        return self._view(self.L.so_decision_scores(self.h), (self.population,), np.float64).copy()

    def enroll_ids(self):
        return self._view(self.L.so_enroll_ids(self.h), (self.cells * 8,), np.int32).copy()

    def enroll_scores(self):
        return self._view(self.L.so_enroll_scores(self.h), (self.cells * 8,), np.float64).copy()

    def winners(self):
        return self._view(self.L.so_winners(self.h), (self.cells,), np.int32).copy()

    def moved_from(self):
        return self._view(self.L.so_moved_from(self.h), (self.cells,), np.int32).copy()

    def moved_to(self):
        return self._view(self.L.so_moved_to(self.h), (self.cells,), np.int32).copy()

    def from_mask(self):
        return np.concatenate([self._view(self.L.so_from_mask(self.h, k), (self.cells,), np.uint8) for k in range(3)])

    def to_mask(self):
        return np.concatenate([self._view(self.L.so_to_mask(self.h, k), (self.cells,), np.uint8) for k in range(3)])

    def plan_entries(self, kind, orientation, sect):
        n = self.L.so_plan_entries(self.h, kind, orientation, sect, None, None, 0)
        dxdy, mag = np.zeros((n, 2), np.int32), np.zeros(n, np.float64)
        self.L.so_plan_entries(self.h, kind, orientation, sect, _p(dxdy), _p(mag), n)
        return dxdy, mag

    def gather_entries(self, kind, sect):
        n = self.L.so_gather_entries(self.h, kind, sect, None, None, None, 0)
        dxdy, mag, mask = np.zeros((n, 2), np.int32), np.zeros(n, np.float64), np.zeros(n, np.uint8)
        self.L.so_gather_entries(self.h, kind, sect, _p(dxdy), _p(mag), _p(mask), n)
        return dxdy, mag, mask
