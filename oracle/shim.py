"""ctypes front end for the flat-C socfield shim (oracle/socfield_shim.h).

TEST INFRASTRUCTURE.  One Python class, `Sim`, drives any build of the shim:

* ``load_ref()``      -> oracle/_ref/libsocfield_ref.so      (unmodified reference, CPU)
* ``load_product()``  -> oracle/build/libsocfield_b200_shim.so (the same shim over the CUDA engine)

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference arm may
import this module with the reference library; the product never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
REF_LIB = os.path.join(HERE, "_ref", "libsocfield_ref.so")
PRODUCT_LIB = os.path.join(HERE, "build", "libsocfield_b200_shim.so")

ERR_NAMES = {1: "IntegrityError", 2: "ConfigError", 3: "ParseError", 4: "SeedingError", 5: "Error"}


class ShimError(RuntimeError):
    def __init__(self, code: int, message: str):
        super().__init__(f"{ERR_NAMES.get(code, code)}: {message}")
        self.code = code
        self.kind = ERR_NAMES.get(code, "Error")
        self.message = message


class EngineCfg(C.Structure):
    _fields_ = [
        ("chunk_k", C.c_int32),
        ("weight_static", C.c_double),
        ("weight_dir_attractive", C.c_double),
        ("weight_dir_repulsive", C.c_double),
        ("weight_recurrent", C.c_double),
        ("goal_bias", C.c_double),
        ("regulation", C.c_int32),
        ("density_radius", C.c_int32),
        ("rebuild_interval", C.c_int64),
        ("rebuild_tolerance", C.c_double),
        ("workers", C.c_int32),
        ("fault_invert_vote_tiebreak", C.c_int32),
    ]


class Field(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("gain", C.c_double), ("decay", C.c_double)]


class Anchor(C.Structure):
    _fields_ = [
        ("kind", C.c_int32),
        ("width", C.c_int32),
        ("height", C.c_int32),
        ("gain", C.c_double),
        ("decay", C.c_double),
        ("x", C.c_int32),
        ("y", C.c_int32),
    ]


class Capture(C.Structure):
    _fields_ = [
        ("decisions", C.c_void_p),
        ("enroll_ids", C.c_void_p),
        ("enroll_scores", C.c_void_p),
        ("winners", C.c_void_p),
        ("moved_from", C.c_void_p),
        ("moved_to", C.c_void_p),
        ("from_mask", C.c_void_p),
        ("to_mask", C.c_void_p),
        ("occupancy_k4", C.c_void_p),
        ("centers_k4", C.c_void_p),
        ("images_k5", C.c_void_p),
        ("phases_seen", C.c_int32),
    ]


def quiet_config(**kw) -> EngineCfg:
    """EngineConfig defaults (reference engine.hpp:108-121) with the unit-test
    fixture's overrides (test_engine.cpp:52-57: workers=1, rebuild_interval=0)."""
    cfg = EngineCfg(8, 1.0, 1.0, 1.0, 1.0, 1.0, 0, 3, 0, 1e-4, 1, 0)
    for k, v in kw.items():
        if not hasattr(cfg, k):
            raise AttributeError(k)
        setattr(cfg, k, v)
    return cfg


def _ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


_LIBS: dict[str, C.CDLL] = {}


def _load(path: str) -> C.CDLL:
    if path in _LIBS:
        return _LIBS[path]
    if not os.path.exists(path):
        raise FileNotFoundError(path)
    lib = C.CDLL(path, mode=C.RTLD_LOCAL)
    vp, cp, sz = C.c_void_p, C.c_char_p, C.c_size_t
    i32, i64, dbl = C.c_int32, C.c_int64, C.c_double
    sig = {
        "shim_impl_name": (cp, []),
        "shim_from_scenario": (C.c_int, [cp, C.c_int, C.POINTER(vp), cp, sz]),
        "shim_from_arrays": (C.c_int, [C.c_int, C.c_int, C.c_int, C.POINTER(EngineCfg), C.POINTER(Field), i64,
                                       vp, vp, vp, vp, vp, vp, vp, C.POINTER(vp), cp, sz]),
        "shim_free": (None, [vp]),
        "shim_set_static_fields": (C.c_int, [vp, i64, C.POINTER(Anchor), cp, sz]),
        "shim_grid": (C.c_int, [vp, C.POINTER(i32), C.POINTER(i32), C.POINTER(i32)]),
        "shim_population": (i64, [vp]),
        "shim_tick_count": (i64, [vp]),
        "shim_set_tick": (None, [vp, i64]),
        "shim_run": (C.c_int, [vp, i64, C.c_int, vp, vp, cp, sz]),
        "shim_tick": (C.c_int, [vp, C.c_int, C.POINTER(i64), cp, sz]),
        "shim_tick_capture": (C.c_int, [vp, C.c_int, C.POINTER(Capture), C.POINTER(i64), cp, sz]),
        "shim_verify": (C.c_int, [vp, cp, sz]),
        "shim_decide": (C.c_int, [vp, i64, C.POINTER(i32), C.POINTER(dbl), C.POINTER(i32), vp, i32, cp, sz]),
        "shim_rebuild_images": (C.c_int, [vp, vp, cp, sz]),
        "shim_plan_entries": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, vp, vp, i32]),
        "shim_plan_fanout": (C.c_int, [vp, C.c_int, C.c_int]),
        "shim_get_centers": (None, [vp, vp]),
        "shim_get_ped_attrs": (None, [vp, vp, vp, vp, vp, vp]),
        "shim_get_occupancy": (None, [vp, vp]),
        "shim_get_image": (None, [vp, C.c_int, vp]),
        "shim_set_centers": (None, [vp, vp]),
        "shim_set_occupancy": (None, [vp, vp]),
        "shim_set_image": (None, [vp, C.c_int, vp]),
        "shim_digest": (C.c_uint64, [vp]),
        "shim_states_identical": (C.c_int, [vp, vp, cp, sz]),
        "shim_clone": (C.c_int, [vp, C.POINTER(vp), cp, sz]),
        "shim_sect_index": (C.c_int, [dbl, dbl]),
        "shim_sort8_desc": (None, [C.POINTER(dbl), C.POINTER(i32)]),
        "shim_multi_step_sum": (dbl, [vp, i64, C.c_int]),
        "shim_strength_at_offset": (None, [C.c_int, C.c_int, C.c_int, dbl, dbl, C.c_int, C.c_int, C.c_int,
                                           C.POINTER(dbl), C.POINTER(dbl)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _LIBS[path] = lib
    return lib


def load_ref() -> C.CDLL:
    return _load(REF_LIB)


def load_product() -> C.CDLL:
    return _load(PRODUCT_LIB)


def have_ref() -> bool:
    return os.path.exists(REF_LIB)


def have_product() -> bool:
    return os.path.exists(PRODUCT_LIB)


@dataclass
class TickCapture:
    decisions: np.ndarray
    enroll_ids: np.ndarray
    enroll_scores: np.ndarray
    winners: np.ndarray
    moved_from: np.ndarray
    moved_to: np.ndarray
    from_mask: np.ndarray
    to_mask: np.ndarray
    occupancy_k4: np.ndarray
    centers_k4: np.ndarray
    images_k5: np.ndarray
    phases_seen: int = 0
    moved: int = 0
    extra: dict = field(default_factory=dict)


class Sim:
    """One (Engine, SimState) pair behind the flat shim."""

    def __init__(self, lib: C.CDLL, handle: int):
        self.lib = lib
        self.h = C.c_void_p(handle)
        w, h, c = C.c_int32(), C.c_int32(), C.c_int32()
        lib.shim_grid(self.h, C.byref(w), C.byref(h), C.byref(c))
        self.width, self.height, self.closed = w.value, h.value, bool(c.value)
        self.cells = self.width * self.height

    # -- construction -----------------------------------------------------
    @staticmethod
    def _check(rc: int, err) -> None:
        if rc != 0:
            raise ShimError(rc, err.value.decode(errors="replace"))

    @classmethod
    def from_scenario(cls, lib: C.CDLL, text: str, workers: int = 1) -> "Sim":
        out = C.c_void_p()
        err = C.create_string_buffer(1024)
        cls._check(lib.shim_from_scenario(text.encode(), workers, C.byref(out), err, len(err)), err)
        return cls(lib, out.value)

    @classmethod
    def from_arrays(cls, lib: C.CDLL, width: int, height: int, peds, *, closed: bool = False,
                    cfg: EngineCfg | None = None, templates=None) -> "Sim":
        """peds: iterable of dicts/tuples (x, y, goal[, fw, fh, period, phase])."""
        cfg = cfg or quiet_config()
        templates = templates or [(7, 7, 1.0, -0.5)] * 3
        tarr = (Field * 3)(*[Field(*t) for t in templates])
        rows = []
        for p in peds:
            if isinstance(p, dict):
                rows.append((p["x"], p["y"], p.get("goal", 0), p.get("fw", 1), p.get("fh", 1),
                             p.get("period", 1), p.get("phase", 0)))
            else:
                p = tuple(p)
                rows.append(p + (0, 1, 1, 1, 0)[len(p) - 2:] if len(p) < 7 else p)
        n = len(rows)
        arr = np.array(rows, dtype=np.int32).reshape(n, 7) if n else np.zeros((0, 7), np.int32)
        cols = [np.ascontiguousarray(arr[:, i]) for i in range(7)]
        cx, cy, goal, fw, fh, period, phase = cols
        out = C.c_void_p()
        err = C.create_string_buffer(1024)
        cls._check(lib.shim_from_arrays(width, height, int(closed), C.byref(cfg), tarr, n, _ptr(cx), _ptr(cy),
                                        _ptr(fw), _ptr(fh), _ptr(period), _ptr(phase), _ptr(goal),
                                        C.byref(out), err, len(err)), err)
        return cls(lib, out.value)

    def clone(self) -> "Sim":
        out = C.c_void_p()
        err = C.create_string_buffer(1024)
        self._check(self.lib.shim_clone(self.h, C.byref(out), err, len(err)), err)
        return Sim(self.lib, out.value)

    def close(self) -> None:
        if self.h:
            self.lib.shim_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- scalar state -------------------------------------------------------
    @property
    def population(self) -> int:
        return self.lib.shim_population(self.h)

    @property
    def tick(self) -> int:
        return self.lib.shim_tick_count(self.h)

    @tick.setter
    def tick(self, value: int) -> None:
        self.lib.shim_set_tick(self.h, value)

    # -- stepping -----------------------------------------------------------
    def run(self, ticks: int, mode: str = "seq", want_phase_us: bool = False):
        moved = np.zeros(max(ticks, 0), np.int64)
        phase = np.zeros((max(ticks, 0), 5), np.int64) if want_phase_us else None
        err = C.create_string_buffer(1024)
        self._check(self.lib.shim_run(self.h, ticks, 0 if mode == "seq" else 1, _ptr(moved), _ptr(phase), err,
                                      len(err)), err)
        return (moved, phase) if want_phase_us else moved

    def step(self, mode: str = "seq") -> int:
        moved = C.c_int64()
        err = C.create_string_buffer(1024)
        self._check(self.lib.shim_tick(self.h, 0 if mode == "seq" else 1, C.byref(moved), err, len(err)), err)
        return moved.value

    def step_capture(self, mode: str = "seq") -> TickCapture:
        c, p = self.cells, self.population
        cap = TickCapture(
            decisions=np.full(p, -9, np.int32),
            enroll_ids=np.full(c * 8, -9, np.int32),
            enroll_scores=np.full(c * 8, np.nan, np.float64),
            winners=np.full(c, -9, np.int32),
            moved_from=np.full(c, -9, np.int32),
            moved_to=np.full(c, -9, np.int32),
            from_mask=np.zeros(3 * c, np.uint8),
            to_mask=np.zeros(3 * c, np.uint8),
            occupancy_k4=np.full(c, -9, np.int32),
            centers_k4=np.full(2 * p, -9, np.int32),
            images_k5=np.zeros(3 * c * 8, np.float32),
        )
        raw = Capture(_ptr(cap.decisions), _ptr(cap.enroll_ids), _ptr(cap.enroll_scores), _ptr(cap.winners),
                      _ptr(cap.moved_from), _ptr(cap.moved_to), _ptr(cap.from_mask), _ptr(cap.to_mask),
                      _ptr(cap.occupancy_k4), _ptr(cap.centers_k4), _ptr(cap.images_k5), 0)
        moved = C.c_int64()
        err = C.create_string_buffer(1024)
        self._check(self.lib.shim_tick_capture(self.h, 0 if mode == "seq" else 1, C.byref(raw), C.byref(moved),
                                               err, len(err)), err)
        cap.phases_seen = raw.phases_seen
        cap.moved = moved.value
        return cap

    def verify(self) -> None:
        err = C.create_string_buffer(1024)
        self._check(self.lib.shim_verify(self.h, err, len(err)), err)

    def decide(self, ped: int):
        d, s, n = C.c_int32(), C.c_double(), C.c_int32()
        cells = np.zeros(2 * 64, np.int32)
        err = C.create_string_buffer(1024)
        self._check(self.lib.shim_decide(self.h, ped, C.byref(d), C.byref(s), C.byref(n), _ptr(cells), 64, err,
                                         len(err)), err)
        return d.value, s.value, [tuple(cells[2 * i:2 * i + 2]) for i in range(min(n.value, 64))]

    def rebuild_images(self) -> np.ndarray:
        out = np.zeros((3, self.height, self.width, 8), np.float32)
        err = C.create_string_buffer(1024)
        self._check(self.lib.shim_rebuild_images(self.h, _ptr(out), err, len(err)), err)
        return out

    def plan_entries(self, kind: int, orientation: int, sect: int):
        n = self.lib.shim_plan_entries(self.h, kind, orientation, sect, None, None, 0)
        dxdy = np.zeros((n, 2), np.int32)
        mag = np.zeros(n, np.float64)
        self.lib.shim_plan_entries(self.h, kind, orientation, sect, _ptr(dxdy), _ptr(mag), n)
        return dxdy, mag

    def plan_fanout(self, kind: int, orientation: int = 0) -> int:
        return self.lib.shim_plan_fanout(self.h, kind, orientation)

    def set_static_fields(self, anchors) -> None:
        """anchors: iterable of (kind 0|1, w, h, gain, decay, x, y)."""
        anchors = list(anchors)
        arr = (Anchor * max(len(anchors), 1))(*[Anchor(*a) for a in anchors])
        err = C.create_string_buffer(1024)
        self._check(self.lib.shim_set_static_fields(self.h, len(anchors), arr, err, len(err)), err)

    # -- arrays -------------------------------------------------------------
    def centers(self) -> np.ndarray:
        out = np.zeros((self.population, 2), np.int32)
        self.lib.shim_get_centers(self.h, _ptr(out))
        return out

    def ped_attrs(self) -> dict:
        p = self.population
        names = ("period", "phase", "goal", "fw", "fh")
        arrs = {k: np.zeros(p, np.int32) for k in names}
        self.lib.shim_get_ped_attrs(self.h, *[_ptr(arrs[k]) for k in names])
        return arrs

    def occupancy(self) -> np.ndarray:
        out = np.zeros((self.height, self.width), np.int32)
        self.lib.shim_get_occupancy(self.h, _ptr(out))
        return out

    def image(self, which: int) -> np.ndarray:
        out = np.zeros((self.height, self.width, 8), np.float32)
        self.lib.shim_get_image(self.h, which, _ptr(out))
        return out

    def images(self) -> np.ndarray:
        return np.stack([self.image(k) for k in range(3)])

    def set_centers(self, xy: np.ndarray) -> None:
        xy = np.ascontiguousarray(xy, np.int32)
        self.lib.shim_set_centers(self.h, _ptr(xy))

    def set_occupancy(self, occ: np.ndarray) -> None:
        occ = np.ascontiguousarray(occ, np.int32)
        self.lib.shim_set_occupancy(self.h, _ptr(occ))

    def set_image(self, which: int, img: np.ndarray) -> None:
        img = np.ascontiguousarray(img, np.float32)
        assert img.size == self.cells * 8
        self.lib.shim_set_image(self.h, which, _ptr(img))

    def digest(self) -> int:
        return int(self.lib.shim_digest(self.h))

    def identical(self, other: "Sim"):
        diag = C.create_string_buffer(1024)
        same = self.lib.shim_states_identical(self.h, other.h, diag, len(diag))
        return bool(same), diag.value.decode(errors="replace")

    def copy_state_from(self, other: "Sim") -> None:
        """Overwrite occupancy, images, centres and tick with another sim's (lockstep mode)."""
        self.set_occupancy(other.occupancy())
        for k in (-1, 0, 1, 2):
            self.set_image(k, other.image(k))
        self.set_centers(other.centers())
        self.tick = other.tick


def fnv1a_digest(occupancy: np.ndarray, images, centers: np.ndarray) -> int:
    """The acceptance digest (acceptance_main.cpp:39-58) recomputed from arrays, in numpy-free Python
    only for small cases; used to cross-check shim_digest."""
    h = 14695981039346656037
    prime = 1099511628211
    mask = (1 << 64) - 1
    blob = occupancy.astype(np.int32).tobytes() + b"".join(np.asarray(i, np.float32).tobytes() for i in images)
    blob += centers.astype(np.int32).tobytes()
    for b in blob:
        h = ((h ^ b) * prime) & mask
    return h
