"""oracle/oracle.py -- TEST INFRASTRUCTURE ONLY.

ctypes front-ends for
  * ``Oracle``    -- the C restatement (oracle/liboracle.so, fewha_oracle.c), and
  * ``RefOracle`` -- the unmodified reference compiled in place
                     (oracle/_ref/libfewha_ref.so, built from ref_shim.cpp).

Both expose the same methods so tests can pin one against the other.  Only
tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this module.
Presets are read with ``load_preset`` which restates the JSON schema of
proj/include/fewha/config_io.hpp:69-179 (defaults included).
"""
from __future__ import annotations

import ctypes as C
import json
import math
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libfewha_ref.so")

ARCSEC = math.pi / (180.0 * 3600.0)

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)


def build(ref: bool = True) -> None:
    """Compile the oracle (and, where /root/reference exists, oracle/_ref)."""
    targets = ["liboracle.so"]
    if ref and os.path.isdir("/root/reference/proj/include"):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


def _ptr(a):
    if a is None:
        return None
    return a.ctypes.data_as(_dp)


def load_preset(path_or_dict) -> dict:
    """JSON preset -> plain dict with every default resolved (config_io.hpp:69-179)."""
    j = path_or_dict
    if not isinstance(j, dict):
        with open(path_or_dict) as f:
            j = json.load(f)
    tel = j["telescope"]
    g = {
        "diameter": float(tel["diameter"]),
        "obstruction_fraction": float(tel.get("obstruction_fraction", 0.0)),
        "obstruction_is_area": 1 if tel.get("obstruction_semantics", "area") == "area" else 0,
        "illumination_threshold": float(tel.get("illumination_threshold", 0.5)),
        "n_subap": [int(w["n_subap"]) for w in j["wfs"]],
        "noise_variance": [float(w["noise_variance"]) for w in j["wfs"]],
        "star_is_lgs": [], "theta_x": [], "theta_y": [], "star_height": [],
        "layer_height": [float(l["height"]) for l in j["layers"]],
        "layer_order": [int(l["grid_order"]) for l in j["layers"]],
        "layer_extent": [float(l.get("extent", 0.0)) for l in j["layers"]],
        "layer_strength": [float(l["relative_strength"]) for l in j["layers"]],
        "n_act": [int(d["n_act"]) for d in j["dms"]],
        "dm_height": [float(d["conjugation_height"]) for d in j["dms"]],
    }
    for s in j["guide_stars"]:
        if "direction_rad" in s:
            tx, ty = s["direction_rad"]
        else:
            tx, ty = (v * ARCSEC for v in s["direction_arcsec"])
        lgs = s["kind"] == "lgs"
        g["star_is_lgs"].append(1 if lgs else 0)
        g["theta_x"].append(float(tx))
        g["theta_y"].append(float(ty))
        g["star_height"].append(float(s["height"]) if lgs else math.inf)
    # L != M projection-fitting extension (not in the reference)
    g["projection"] = 1 if j.get("fitting", "identity") == "projection" else 0
    g["dm_theta_x"], g["dm_theta_y"], g["dm_layer_mask"], g["dm_extent_in"] = [], [], [], []
    for d in j["dms"]:
        if "direction_rad" in d:
            tx, ty = d["direction_rad"]
        elif "direction_arcsec" in d:
            tx, ty = (v * ARCSEC for v in d["direction_arcsec"])
        else:
            tx = ty = 0.0
        g["dm_theta_x"].append(float(tx))
        g["dm_theta_y"].append(float(ty))
        g["dm_layer_mask"].append(sum(1 << int(l) for l in d.get("layers", [])))
        g["dm_extent_in"].append(float(d.get("extent", 0.0)))
    sol = j["solver"]
    g.update(
        pcg_max_iter=int(sol["pcg_max_iter"]),
        pcg_tolerance=float(sol.get("pcg_tolerance", 0.0)),
        alpha=float(sol["alpha"]),
        wavelet_order=int(sol.get("wavelet_order", 3)),
        outer_scale=float(sol.get("outer_scale", 25.0)),
        spectral_exponent=float(sol.get("spectral_exponent", 11.0 / 6.0)),
        precond_mode={"exact": 0, "approximate": 1, "balanced": 2}[sol.get("preconditioner", "approximate")],
        precond_coarse_weight=float(sol.get("precond_coarse_weight", 4.0)),
        precond_balance_exponent=float(sol.get("precond_balance_exponent", 0.5)),
        dense_size_cap=int(sol.get("dense_size_cap", 20000)),
        fault_sh_adjoint=1 if sol.get("fault", "") == "sh_adjoint" else 0,
        loop_closed=1 if j["loop"]["mode"] == "closed" else 0,
        gain=float(j["loop"]["gain"]),
    )
    return g


class _Cfg(C.Structure):
    _fields_ = [
        ("diameter", C.c_double), ("obstruction_fraction", C.c_double), ("illumination_threshold", C.c_double),
        ("obstruction_is_area", C.c_int), ("n_wfs", C.c_int), ("n_subap", _ip), ("noise_variance", _dp),
        ("star_is_lgs", _ip), ("theta_x", _dp), ("theta_y", _dp), ("star_height", _dp),
        ("n_layers", C.c_int), ("layer_height", _dp), ("layer_order", _ip), ("layer_extent", _dp),
        ("layer_strength", _dp), ("n_dms", C.c_int), ("n_act", _ip), ("dm_height", _dp),
        ("pcg_max_iter", C.c_int), ("pcg_tolerance", C.c_double), ("alpha", C.c_double),
        ("wavelet_order", C.c_int), ("outer_scale", C.c_double), ("spectral_exponent", C.c_double),
        ("precond_mode", C.c_int), ("precond_coarse_weight", C.c_double),
        ("precond_balance_exponent", C.c_double), ("dense_size_cap", C.c_longlong),
        ("fault_sh_adjoint", C.c_int), ("loop_closed", C.c_int), ("gain", C.c_double),
        ("projection", C.c_int), ("dm_theta_x", _dp), ("dm_theta_y", _dp), ("dm_layer_mask", _ip),
        ("dm_extent_in", _dp),
    ]


@dataclass
class Dims:
    n: int
    S: int
    A: int
    L: int
    W: int
    M: int
    iters: int
    Nw: int


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class _Base:
    """Shared numpy-facing API (same method names on both back-ends)."""

    def _chk(self, rc):
        if rc:
            raise OracleError(rc, self.last_error())

    def geometry(self):
        d = self.dims
        ext = np.zeros(d.L)
        dext = np.zeros(d.M)
        masks = np.zeros(sum(n * n for n in self.n_subap), np.uint8)
        self._geometry(ext, dext, masks)
        return ext, dext, masks

    def wavelet(self, x, inverse):
        y = np.array(x, np.float64, copy=True)
        self._chk(self._lib_wavelet(self.h, 1 if inverse else 0, _ptr(y)))
        return y

    def _unary(self, fn, x, nout):
        x = np.ascontiguousarray(x, np.float64)
        y = np.zeros(nout)
        self._chk(fn(self.h, _ptr(x), _ptr(y)))
        return y

    def preconditioner(self):
        out = np.zeros(self.dims.n)
        self._precond(self.h, _ptr(out))
        return out

    def step(self, meas):
        d = self.dims
        meas = np.ascontiguousarray(meas, np.float64)
        c = np.zeros(d.n)
        a = np.zeros(d.A)
        rho = np.zeros(max(d.iters, 1))
        nr = C.c_int(0)
        self._chk(self._step(meas, c, a, rho, nr))
        return c, a, rho[: nr.value].copy()

    def get_state(self):
        d = self.dims
        st = {k: np.zeros(d.n) for k in ("c", "b", "r", "p", "q")}
        st["scalars"] = np.zeros(3)
        st["a_prev2"] = np.zeros(d.A)
        st["a_prev"] = np.zeros(d.A)
        self._get_state(self.h, *(_ptr(st[k]) for k in ("c", "b", "r", "p", "q", "scalars", "a_prev2", "a_prev")))
        return st

    def set_state(self, st):
        arrs = [np.ascontiguousarray(st[k], np.float64) for k in ("c", "b", "r", "p", "q", "scalars", "a_prev2", "a_prev")]
        self._set_state(self.h, *(_ptr(a) for a in arrs))

    def apply_M(self, x):
        return self._unary(self._lib.__getattr__(self._p + "apply_M"), x, self.dims.n)

    def build_rhs(self, meas):
        return self._unary(self._lib.__getattr__(self._p + "build_rhs"), meas, self.dims.n)

    def fit(self, c):
        return self._unary(self._lib.__getattr__(self._p + "fit"), c, self.dims.A)

    def propagate(self, layers):
        return self._unary(self._lib.__getattr__(self._p + "propagate"), layers, self.dims.Nw)

    def propagate_transpose(self, wf):
        return self._unary(self._lib.__getattr__(self._p + "propagate_transpose"), wf, self.dims.n)

    def sh(self, wf):
        return self._unary(self._lib.__getattr__(self._p + "sh"), wf, self.dims.S)

    def sh_transpose(self, meas):
        return self._unary(self._lib.__getattr__(self._p + "sh_transpose"), meas, self.dims.Nw)

    def add_dm_slopes(self, a, meas):
        m = np.array(meas, np.float64, copy=True)
        a = np.ascontiguousarray(a, np.float64)
        self._chk(self._lib.__getattr__(self._p + "add_dm_slopes")(self.h, _ptr(a), _ptr(m)))
        return m

    def build_preconditioner(self):
        self._chk(self._lib.__getattr__(self._p + "build_preconditioner")(self.h))


class Oracle(_Base):
    """The C restatement (fewha_oracle.c)."""

    _p = "orc_"

    def __init__(self, preset, loop_mode=None, gain=None, overrides=None):
        lib = C.CDLL(ORACLE_SO)
        self._lib = lib
        lib.orc_create.restype = C.c_void_p
        lib.orc_create.argtypes = [C.POINTER(_Cfg), C.c_char_p, C.c_int, _ip]
        lib.orc_last_error.restype = C.c_char_p
        lib.orc_last_error.argtypes = [C.c_void_p]
        for name in ("apply_M", "build_rhs", "fit", "propagate", "propagate_transpose", "sh", "sh_transpose",
                     "add_dm_slopes", "wavelet", "build_preconditioner", "step", "reset", "dims", "geometry",
                     "get_state", "set_state", "preconditioner", "destroy"):
            getattr(lib, "orc_" + name).argtypes = None
        g = load_preset(preset) if not isinstance(preset, dict) or "diameter" not in preset else dict(preset)
        if loop_mode is not None:
            g["loop_closed"] = 1 if loop_mode == "closed" else 0
        if gain is not None:
            g["gain"] = float(gain)
        if overrides:
            g.update(overrides)
        self.g = g
        self.n_subap = g["n_subap"]
        keep = {}

        def arr(name, ct):
            a = (ct * len(g[name]))(*g[name])
            keep[name] = a
            return a

        cfg = _Cfg(
            g["diameter"], g["obstruction_fraction"], g["illumination_threshold"], g["obstruction_is_area"],
            len(g["n_subap"]), arr("n_subap", C.c_int), arr("noise_variance", C.c_double),
            arr("star_is_lgs", C.c_int), arr("theta_x", C.c_double), arr("theta_y", C.c_double),
            arr("star_height", C.c_double), len(g["layer_height"]), arr("layer_height", C.c_double),
            arr("layer_order", C.c_int), arr("layer_extent", C.c_double), arr("layer_strength", C.c_double),
            len(g["n_act"]), arr("n_act", C.c_int), arr("dm_height", C.c_double), g["pcg_max_iter"],
            g["pcg_tolerance"], g["alpha"], g["wavelet_order"], g["outer_scale"], g["spectral_exponent"],
            g["precond_mode"], g["precond_coarse_weight"], g["precond_balance_exponent"], g["dense_size_cap"],
            g["fault_sh_adjoint"], g["loop_closed"], g["gain"],
            g["projection"], arr("dm_theta_x", C.c_double), arr("dm_theta_y", C.c_double),
            arr("dm_layer_mask", C.c_int), arr("dm_extent_in", C.c_double),
        )
        err = C.create_string_buffer(512)
        code = C.c_int(0)
        h = lib.orc_create(C.byref(cfg), err, 512, C.byref(code))
        if not h:
            raise OracleError(code.value, err.value.decode())
        self.h = C.c_void_p(h)
        d = (C.c_longlong * 8)()
        lib.orc_dims(self.h, d)
        self.dims = Dims(*[int(v) for v in d])
        self._lib_wavelet = lib.orc_wavelet
        self._precond = lib.orc_preconditioner
        self._get_state = lib.orc_get_state
        self._set_state = lib.orc_set_state

    def last_error(self):
        return self._lib.orc_last_error(self.h).decode()

    def _geometry(self, ext, dext, masks):
        self._lib.orc_geometry(self.h, _ptr(ext), _ptr(dext), masks.ctypes.data_as(C.c_void_p))

    def _step(self, meas, c, a, rho, nr):
        return self._lib.orc_step(self.h, _ptr(meas), _ptr(c), _ptr(a), _ptr(rho), C.byref(nr))

    def reset(self):
        self._lib.orc_reset(self.h)

    def __del__(self):
        try:
            self._lib.orc_destroy(self.h)
        except Exception:
            pass

    @staticmethod
    def wavelet_grid(order, x, inverse):
        lib = C.CDLL(ORACLE_SO)
        y = np.array(x, np.float64, copy=True)
        rc = lib.orc_wavelet_grid(C.c_int(order), C.c_int(y.shape[0]), C.c_int(1 if inverse else 0), _ptr(y))
        if rc:
            raise OracleError(rc, "wavelet_grid: bad arguments")
        return y


class RefOracle(_Base):
    """The unmodified reference, compiled in place (oracle/_ref/libfewha_ref.so)."""

    _p = "ref_"

    @staticmethod
    def available():
        return os.path.exists(REF_SO)

    def __init__(self, preset_path, threads=0, loop_mode=None, gain=None):
        lib = C.CDLL(REF_SO)
        self._lib = lib
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_create.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_double, C.POINTER(C.c_void_p)]
        lib.ref_synthesize.argtypes = [C.c_void_p, C.c_ulonglong, C.c_int, _dp, _dp]
        lib.ref_record.argtypes = [C.c_void_p, C.c_ulonglong, C.c_int, C.c_int, _dp, _dp, _dp, _dp, _dp]
        lib.ref_atmosphere.argtypes = [C.c_void_p, C.c_ulonglong, _dp]
        h = C.c_void_p()
        lm = -1 if loop_mode is None else (0 if loop_mode == "closed" else 1)
        rc = lib.ref_create(str(preset_path).encode(), threads, lm, -1.0 if gain is None else float(gain), C.byref(h))
        if rc:
            raise OracleError(rc, lib.ref_last_error().decode())
        self.h = h
        d = (C.c_longlong * 9)()
        lib.ref_dims(self.h, d)
        self.dims = Dims(*[int(v) for v in d[:8]])
        self.threads = int(d[8])
        self.n_subap = load_preset(preset_path)["n_subap"]
        self._lib_wavelet = lib.ref_wavelet
        self._precond = lib.ref_preconditioner
        self._get_state = lib.ref_get_state
        self._set_state = lib.ref_set_state

    def last_error(self):
        return self._lib.ref_last_error().decode()

    def _geometry(self, ext, dext, masks):
        self._lib.ref_geometry(self.h, _ptr(ext), _ptr(dext), masks.ctypes.data_as(C.c_void_p))

    def _step(self, meas, c, a, rho, nr):
        return self._lib.ref_step(self.h, _ptr(meas), _ptr(c), _ptr(a), _ptr(rho), C.byref(nr), None)

    def reset(self):
        self._lib.ref_reset(self.h)

    def __del__(self):
        try:
            self._lib.ref_destroy(self.h)
        except Exception:
            pass

    def atmosphere(self, seed):
        out = np.zeros(self.dims.n)
        self._chk(self._lib.ref_atmosphere(self.h, seed, _ptr(out)))
        return out

    def synthesize(self, seed, k, a_prev2=None):
        out = np.zeros(self.dims.S)
        a = None if a_prev2 is None else np.ascontiguousarray(a_prev2, np.float64)
        self._chk(self._lib.ref_synthesize(self.h, seed, k, _ptr(a), _ptr(out)))
        return out

    def record(self, seed, frames, k0=0):
        """Closed loop exactly as run_bench (bench.hpp:144-154): per frame the slopes
        fed to step, and the step's c, a^(1), rho, wall time."""
        d = self.dims
        meas = np.zeros((frames, d.S))
        c = np.zeros((frames, d.n))
        a = np.zeros((frames, d.A))
        rho = np.zeros((frames, d.iters))
        us = np.zeros(frames)
        self._chk(self._lib.ref_record(self.h, seed, k0, frames, _ptr(meas), _ptr(c), _ptr(a), _ptr(rho), _ptr(us)))
        return meas, c, a, rho, us

    def truth_at_step(self, seed, k):
        out = np.zeros(self.dims.n)
        self._chk(self._lib.ref_truth_at_step(self.h, C.c_ulonglong(seed), C.c_int(k), _ptr(out)))
        return out

    def quality(self, layers, dm):
        """evaluate_quality: (field_rms, layer_rel_err, rms_per_dir)."""
        out = np.zeros(2 + 4096)
        lay = np.ascontiguousarray(layers, np.float64)
        a = np.ascontiguousarray(dm, np.float64)
        self._chk(self._lib.ref_quality(self.h, _ptr(lay), _ptr(a), _ptr(out)))
        return out[0], out[1], out[2:]

    def run_closed_loop(self, n_steps, atm=1, noise=2, threads=0):
        d = self.dims
        fr, le = np.zeros(n_steps), np.zeros(n_steps)
        rho = np.zeros((n_steps, d.iters))
        o2 = np.zeros(2)
        self._chk(self._lib.ref_run_closed_loop(self.h, C.c_int(n_steps), C.c_ulonglong(atm), C.c_ulonglong(noise),
                                                C.c_int(threads), _ptr(fr), _ptr(le), _ptr(rho), _ptr(o2)))
        return {"field_rms": fr, "layer_rel_err": le, "rho": rho, "uncorrected_field_rms": o2[0],
                "final_field_rms": o2[1]}

    @staticmethod
    def gauss(seed, count):
        lib = C.CDLL(REF_SO)
        out = np.zeros(count)
        rc = lib.ref_gauss(C.c_ulonglong(seed), C.c_int(count), _ptr(out))
        if rc:
            raise OracleError(rc, lib.ref_last_error().decode())
        return out

    def time_steps(self, meas_stream, frames):
        ms = np.ascontiguousarray(meas_stream, np.float64).reshape(-1, self.dims.S)
        us = np.zeros(frames)
        self._chk(self._lib.ref_time_steps(self.h, _ptr(ms), C.c_int(ms.shape[0]), C.c_int(frames), _ptr(us)))
        return us

    @staticmethod
    def wavelet_grid(order, x, inverse):
        lib = C.CDLL(REF_SO)
        y = np.array(x, np.float64, copy=True)
        rc = lib.ref_wavelet_grid(C.c_int(order), C.c_int(y.shape[0]), C.c_int(1 if inverse else 0), _ptr(y))
        if rc:
            raise OracleError(rc, lib.ref_last_error().decode())
        return y


def rel_err(a, b) -> float:
    """||a-b|| / max(||a||, ||b||), 0 when both vanish (grid.hpp:88-98)."""
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    ref = math.sqrt(max(float(a @ a), float(b @ b)))
    return 0.0 if ref == 0.0 else float(np.linalg.norm(a - b)) / ref
