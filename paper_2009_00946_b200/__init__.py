"""B200-native FEWHA tomographic reconstructor (arXiv 2009.00946).

Python mirror of the reference's C++ solver API (proj/include/fewha/
reconstructor.hpp) over the C-ABI in include/fewha_gpu.h.  The compute path
is the sm_100a library ``lib/libfewha_gpu.so``; there is no CPU fallback --
importing works without a GPU, but constructing a Reconstructor fails loudly
when the library or a CUDA device is missing.

    rec = Reconstructor("presets/elt_mcao84.json", precision=64)
    rec.build_preconditioner()                 # Reconstructor::build_preconditioner
    a1 = rec.step(slopes)                      # Reconstructor::step -> a^(1)
    rec.last_rho, rec.coeffs()                 # last_telemetry().rho, st.c
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libfewha_gpu.so")

FEWHA_OK, FEWHA_RUNTIME, FEWHA_CONFIG, FEWHA_ARG = 0, 1, 2, 3

# every entry point declared in include/fewha_gpu.h
EXPORTS = (
    "fewha_gpu_create", "fewha_gpu_create_from_json", "fewha_gpu_override_loop", "fewha_gpu_create_error",
    "fewha_gpu_last_error", "fewha_gpu_destroy", "fewha_gpu_dims", "fewha_gpu_preset_info", "fewha_gpu_geometry",
    "fewha_gpu_build_preconditioner", "fewha_gpu_preconditioner", "fewha_gpu_step", "fewha_gpu_reset",
    "fewha_gpu_get_state", "fewha_gpu_set_state", "fewha_gpu_set_stream", "fewha_gpu_device_buffers",
    "fewha_gpu_load_slopes", "fewha_gpu_step_device", "fewha_gpu_sync", "fewha_gpu_launches_per_step", "fewha_gpu_profile_step", "fewha_gpu_phase_stamps", "fewha_gpu_apply_M",
    "fewha_gpu_build_rhs", "fewha_gpu_add_dm_slopes", "fewha_gpu_fit_to_mirrors", "fewha_gpu_wavelet",
    "fewha_gpu_propagate", "fewha_gpu_propagate_transpose", "fewha_gpu_sh", "fewha_gpu_sh_transpose",
    "fewha_gpu_forward_slopes", "fewha_gpu_shard_range", "fewha_gpu_nccl_unique_id", "fewha_gpu_shard",
    "fewha_gpu_shard_wfs", "fewha_gpu_group_step_device", "fewha_gpu_enable_telemetry", "fewha_gpu_last_telemetry",
    "fewha_gpu_wfs_operator", "fewha_gpu_plan_info", "fewha_gpu_last_launch_times",
    "fewha_gpu_sim_quality_size", "fewha_gpu_sim_atmosphere", "fewha_gpu_sim_synthesize", "fewha_gpu_sim_quality",
    "fewha_gpu_run_closed_loop", "fewha_gpu_sim_gauss", "fewha_gpu_create_multi",
)


class FewhaError(RuntimeError):
    """Runtime failure (reference: std::runtime_error, CLI exit 1)."""

    code = FEWHA_RUNTIME


class ConfigError(FewhaError):
    """Configuration error (reference: fewha::config_error, CLI exit 2)."""

    code = FEWHA_CONFIG


class ArgumentError(FewhaError, ValueError):
    """Bad argument / size mismatch (reference: std::invalid_argument)."""

    code = FEWHA_ARG


_ERR = {FEWHA_RUNTIME: FewhaError, FEWHA_CONFIG: ConfigError, FEWHA_ARG: ArgumentError}


class _Dims(C.Structure):
    _fields_ = [("n_coeff", C.c_longlong), ("n_slopes", C.c_longlong), ("n_act", C.c_longlong),
                ("n_wavefront", C.c_longlong), ("n_layers", C.c_int), ("n_wfs", C.c_int), ("n_dms", C.c_int),
                ("pcg_iters", C.c_int), ("batch", C.c_int), ("precision", C.c_int)]


class _State(C.Structure):
    _fields_ = [("c", C.POINTER(C.c_double)), ("b", C.POINTER(C.c_double)), ("r", C.POINTER(C.c_double)),
                ("p", C.POINTER(C.c_double)), ("q", C.POINTER(C.c_double)), ("scalars", C.c_double * 3),
                ("a_prev2", C.POINTER(C.c_double)), ("a_prev", C.POINTER(C.c_double))]


class _Telemetry(C.Structure):
    _fields_ = [("step", C.c_longlong), ("valid", C.c_int), ("stage1_us", C.c_double), ("stage2_us", C.c_double),
                ("stage3_us", C.c_double), ("pcg_us", C.c_double), ("fit_us", C.c_double), ("total_us", C.c_double)]


class _Plan(C.Structure):
    _fields_ = [(k, C.c_int) for k in ("cluster_ctas", "tail", "gather_rows", "gather_ctas_per_sm", "inverse_staged",
                                       "wfs_ctas_per_sm", "wfs_tiles", "launches_per_step", "whole_layer",
                                       "gather_instances", "wfs_instances", "gather_direct")]


class _DevBufs(C.Structure):
    _fields_ = [("slopes", C.c_void_p), ("coeffs", C.c_void_p), ("dm", C.c_void_p), ("rho", C.c_void_p),
                ("status", C.c_void_p), ("n_rho", C.c_void_p)]


_lib_handle = None


def build(verbose: bool = False) -> str:
    """Compile the sm_100a library in-tree (nvcc -gencode arch=compute_100a,code=sm_100a)."""
    out = subprocess.run(["make", "-C", HERE, "-s"], capture_output=not verbose, text=True)
    if out.returncode != 0:
        raise RuntimeError("building libfewha_gpu.so failed:\n" + (out.stdout or "") + (out.stderr or ""))
    return LIB_PATH


def lib() -> C.CDLL:
    """Load the native library; raises if it has not been built (no fallback)."""
    global _lib_handle
    if _lib_handle is None:
        if not os.path.exists(LIB_PATH):
            raise FewhaError(f"native library missing: {LIB_PATH} (run paper_2009_00946_b200.build())")
        L = C.CDLL(LIB_PATH)
        dp = C.POINTER(C.c_double)
        vp = C.c_void_p
        L.fewha_gpu_create.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, C.POINTER(vp)]
        L.fewha_gpu_create_from_json.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, C.POINTER(vp)]
        L.fewha_gpu_create_multi.argtypes = [C.c_char_p, C.c_int, C.c_int, C.POINTER(C.c_int), C.c_int, C.POINTER(vp)]
        L.fewha_gpu_create_error.restype = C.c_char_p
        L.fewha_gpu_last_error.restype = C.c_char_p
        L.fewha_gpu_last_error.argtypes = [vp]
        L.fewha_gpu_destroy.argtypes = [vp]
        L.fewha_gpu_override_loop.argtypes = [vp, C.c_int, C.c_double]
        L.fewha_gpu_dims.argtypes = [vp, C.POINTER(_Dims)]
        L.fewha_gpu_geometry.argtypes = [vp, dp, dp, C.c_void_p]
        L.fewha_gpu_preset_info.argtypes = [C.c_char_p, C.POINTER(_Dims), dp, dp, C.c_void_p]
        L.fewha_gpu_build_preconditioner.argtypes = [vp]
        L.fewha_gpu_preconditioner.argtypes = [vp, dp]
        L.fewha_gpu_step.argtypes = [vp, dp, dp, dp, dp, C.POINTER(C.c_int)]
        L.fewha_gpu_reset.argtypes = [vp]
        L.fewha_gpu_get_state.argtypes = [vp, C.c_int, C.POINTER(_State)]
        L.fewha_gpu_set_state.argtypes = [vp, C.c_int, C.POINTER(_State)]
        L.fewha_gpu_set_stream.argtypes = [vp, vp]
        L.fewha_gpu_device_buffers.argtypes = [vp, C.POINTER(_DevBufs)]
        L.fewha_gpu_step_device.argtypes = [vp, vp]
        L.fewha_gpu_load_slopes.argtypes = [vp, vp, C.c_int]
        L.fewha_gpu_sync.argtypes = [vp]
        L.fewha_gpu_launches_per_step.argtypes = [vp]
        L.fewha_gpu_profile_step.argtypes = [vp, C.POINTER(C.c_float), C.POINTER(C.c_int), C.c_int]
        L.fewha_gpu_phase_stamps.argtypes = [vp, C.c_void_p, C.c_longlong]
        for name in ("apply_M", "build_rhs", "add_dm_slopes", "fit_to_mirrors", "propagate",
                     "propagate_transpose", "sh", "sh_transpose"):
            getattr(L, "fewha_gpu_" + name).argtypes = [vp, dp, dp, C.c_int]
        L.fewha_gpu_wavelet.argtypes = [vp, C.c_int, dp, C.c_int]
        L.fewha_gpu_forward_slopes.argtypes = [vp, dp, dp, dp, C.c_int]
        L.fewha_gpu_wfs_operator.argtypes = [vp, C.c_int, dp, dp, dp, C.c_int]
        L.fewha_gpu_plan_info.argtypes = [vp, C.POINTER(_Plan)]
        L.fewha_gpu_last_launch_times.argtypes = [vp, C.POINTER(C.c_float), C.POINTER(C.c_int), C.c_int]
        u64 = C.c_ulonglong
        L.fewha_gpu_sim_quality_size.argtypes = [vp]
        L.fewha_gpu_sim_gauss.argtypes = [C.c_int, u64, C.c_int, dp]
        L.fewha_gpu_sim_atmosphere.argtypes = [vp, u64, C.c_int, dp]
        L.fewha_gpu_sim_synthesize.argtypes = [vp, dp, dp, u64, dp]
        L.fewha_gpu_sim_quality.argtypes = [vp, dp, dp, dp]
        L.fewha_gpu_run_closed_loop.argtypes = [vp, C.c_int, u64, u64, dp, dp, dp]
        ip = C.POINTER(C.c_int)
        L.fewha_gpu_shard_range.argtypes = [C.c_char_p, C.c_int, C.c_int, ip, ip]
        L.fewha_gpu_nccl_unique_id.argtypes = [C.c_char_p]
        L.fewha_gpu_shard.argtypes = [vp, C.c_int, C.c_int, C.c_char_p]
        L.fewha_gpu_shard_wfs.argtypes = [vp, ip, ip]
        L.fewha_gpu_group_step_device.argtypes = [C.POINTER(vp), C.c_int]
        L.fewha_gpu_enable_telemetry.argtypes = [vp, C.c_int]
        L.fewha_gpu_last_telemetry.argtypes = [vp, C.POINTER(_Telemetry)]
        _lib_handle = L
    return _lib_handle


def _dp(a):
    return None if a is None else a.ctypes.data_as(C.POINTER(C.c_double))


def _f64(a, n=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if n is not None and a.size != n:
        raise ArgumentError(f"expected {n} values, got {a.size}")
    return a


def _raise_create(rc):
    if rc != FEWHA_OK:
        raise _ERR.get(rc, FewhaError)(lib().fewha_gpu_create_error().decode())


def shard_range(preset, rank: int, world: int) -> tuple[int, int]:
    """WFS range [begin, end) owned by shard rank/world (host only, no device):
    contiguous ranges minimising the largest per-shard wavefront node count."""
    b, e = C.c_int(), C.c_int()
    _raise_create(lib().fewha_gpu_shard_range(os.fspath(preset).encode(), rank, world, C.byref(b), C.byref(e)))
    return b.value, e.value


def nccl_unique_id() -> bytes:
    """A fresh 128-byte ncclUniqueId (rank 0 makes it, every rank passes it to shard())."""
    buf = C.create_string_buffer(128)
    _raise_create(lib().fewha_gpu_nccl_unique_id(buf))
    return buf.raw


def group_step_device(members) -> None:
    """One frame of an in-process shard group (members[r] is shard r of len(members))."""
    arr = (C.c_void_p * len(members))(*[m._h for m in members])
    rc = lib().fewha_gpu_group_step_device(arr, len(members))
    if rc != FEWHA_OK:
        raise _ERR.get(rc, FewhaError)(lib().fewha_gpu_last_error(members[0]._h).decode())


@dataclass
class Dims:
    n: int      # wavelet coefficients (CoeffLayout total)
    S: int      # slopes (MeasurementLayout total)
    A: int      # actuators
    Nw: int     # wavefront nodes
    L: int
    W: int
    M: int
    iters: int
    batch: int
    precision: int


class Reconstructor:
    """Drop-in for fewha::Reconstructor + its ReconstructorState (device resident).

    precision: 64 (parity mode, 1e-9) or 32 (1e-4).  batch: independent
    instances stepped together; per-frame arrays are then [batch, ...]."""

    def __init__(self, preset, precision: int = 64, batch: int = 1, device: int = 0, loop_mode=None, gain=None,
                 devices=None):
        """devices: a list of CUDA ordinals (fewha_gpu_create_multi): more than one makes
        the handle an in-process per-WFS shard group stepped as one reconstructor."""
        L = lib()
        h = C.c_void_p()
        if devices is not None:
            arr = (C.c_int * len(devices))(*devices)
            rc = L.fewha_gpu_create_multi(os.fspath(preset).encode(), precision, batch, arr, len(devices), C.byref(h))
        elif isinstance(preset, dict):
            import json
            rc = L.fewha_gpu_create_from_json(json.dumps(preset).encode(), precision, batch, device, C.byref(h))
        else:
            rc = L.fewha_gpu_create(os.fspath(preset).encode(), precision, batch, device, C.byref(h))
        if rc:
            raise _ERR.get(rc, FewhaError)(L.fewha_gpu_create_error().decode())
        self._h = h
        self._L = L
        d = _Dims()
        self._chk(L.fewha_gpu_dims(h, C.byref(d)))
        self.dims = Dims(d.n_coeff, d.n_slopes, d.n_act, d.n_wavefront, d.n_layers, d.n_wfs, d.n_dms, d.pcg_iters,
                         d.batch, d.precision)
        if loop_mode is not None or gain is not None:
            self.override_loop(loop_mode, gain)
        self.last_rho = None
        self._last_c = None

    # -- plumbing --------------------------------------------------------------
    def _chk(self, rc):
        if rc:
            raise _ERR.get(rc, FewhaError)(self._L.fewha_gpu_last_error(self._h).decode())

    def close(self):
        if getattr(self, "_h", None):
            self._L.fewha_gpu_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def override_loop(self, loop_mode=None, gain=None):
        lm = -1 if loop_mode is None else (0 if loop_mode == "closed" else 1)
        self._chk(self._L.fewha_gpu_override_loop(self._h, lm, -1.0 if gain is None else float(gain)))

    # -- reference API -------------------------------------------------------------
    def geometry(self):
        d = self.dims
        ext, dext = np.zeros(d.L), np.zeros(d.M)
        masks = np.zeros((d.S // 2,), np.uint8)
        self._chk(self._L.fewha_gpu_geometry(self._h, _dp(ext), _dp(dext), masks.ctypes.data_as(C.c_void_p)))
        return ext, dext, masks

    def build_preconditioner(self):
        self._chk(self._L.fewha_gpu_build_preconditioner(self._h))

    def preconditioner(self):
        out = np.zeros(self.dims.n)
        self._chk(self._L.fewha_gpu_preconditioner(self._h, _dp(out)))
        return out

    def step(self, slopes, want_coeffs: bool = True):
        """Reconstructor::step: returns a^(1) ([A] or [batch, A]); st.c via coeffs()."""
        d = self.dims
        s = _f64(slopes, d.S * d.batch)
        a = np.zeros(d.A * d.batch)
        c = np.zeros(d.n * d.batch) if want_coeffs else None
        rho = np.zeros(d.iters * d.batch)
        nr = (C.c_int * d.batch)()
        self._chk(self._L.fewha_gpu_step(self._h, _dp(s), _dp(c), _dp(a), _dp(rho), nr))
        rho = rho.reshape(d.batch, d.iters)
        self.last_rho = [rho[b, : nr[b]].copy() for b in range(d.batch)]
        self._last_c = c
        if d.batch == 1:
            self.last_rho = self.last_rho[0]
            return a
        return a.reshape(d.batch, d.A)

    def coeffs(self):
        """st.c after the last step."""
        if self._last_c is None:
            return self.get_state()["c"]
        c = self._last_c
        return c if self.dims.batch == 1 else c.reshape(self.dims.batch, self.dims.n)

    def reset(self):
        self._chk(self._L.fewha_gpu_reset(self._h))
        self._last_c = None

    def get_state(self, instance: int = 0):
        d = self.dims
        st = {k: np.zeros(d.n) for k in ("c", "b", "r", "p", "q")}
        st["a_prev2"] = np.zeros(d.A)
        st["a_prev"] = np.zeros(d.A)
        cs = _State(*(_dp(st[k]) for k in ("c", "b", "r", "p", "q")), (C.c_double * 3)(), _dp(st["a_prev2"]),
                    _dp(st["a_prev"]))
        self._chk(self._L.fewha_gpu_get_state(self._h, instance, C.byref(cs)))
        st["scalars"] = np.array(list(cs.scalars))
        return st

    def set_state(self, st, instance: int = 0):
        d = self.dims
        arr = {k: _f64(st[k], d.n) for k in ("c", "b", "r", "p", "q")}
        arr["a_prev2"] = _f64(st["a_prev2"], d.A)
        arr["a_prev"] = _f64(st["a_prev"], d.A)
        sc = (C.c_double * 3)(*[float(x) for x in st["scalars"]])
        cs = _State(*(_dp(arr[k]) for k in ("c", "b", "r", "p", "q")), sc, _dp(arr["a_prev2"]), _dp(arr["a_prev"]))
        self._chk(self._L.fewha_gpu_set_state(self._h, instance, C.byref(cs)))
        self._last_c = None

    # -- operator entry points (count = stacked inputs) -------------------------------
    def _op(self, fn, x, nin, nout, *extra):
        x = _f64(x)
        count = x.size // nin
        if count * nin != x.size or count < 1:
            raise ArgumentError(f"input size {x.size} is not a multiple of {nin}")
        out = np.zeros(count * nout)
        self._chk(fn(self._h, _dp(x), _dp(out), count, *extra))
        return out if count == 1 else out.reshape(count, nout)

    def apply_M(self, x):
        return self._op(self._L.fewha_gpu_apply_M, x, self.dims.n, self.dims.n)

    def build_rhs(self, meas):
        return self._op(self._L.fewha_gpu_build_rhs, meas, self.dims.S, self.dims.n)

    def fit(self, c):
        return self._op(self._L.fewha_gpu_fit_to_mirrors, c, self.dims.n, self.dims.A)

    def propagate(self, layers):
        return self._op(self._L.fewha_gpu_propagate, layers, self.dims.n, self.dims.Nw)

    def propagate_transpose(self, wf):
        return self._op(self._L.fewha_gpu_propagate_transpose, wf, self.dims.Nw, self.dims.n)

    def sh(self, wf):
        return self._op(self._L.fewha_gpu_sh, wf, self.dims.Nw, self.dims.S)

    def sh_transpose(self, meas):
        return self._op(self._L.fewha_gpu_sh_transpose, meas, self.dims.S, self.dims.Nw)

    def wavelet(self, x, inverse: bool):
        y = np.array(_f64(x), copy=True)
        count = y.size // self.dims.n
        self._chk(self._L.fewha_gpu_wavelet(self._h, 1 if inverse else 0, _dp(y), count))
        return y

    def add_dm_slopes(self, a, meas):
        m = np.array(_f64(meas), copy=True)
        a = _f64(a)
        count = m.size // self.dims.S
        self._chk(self._L.fewha_gpu_add_dm_slopes(self._h, _dp(a), _dp(m), count))
        return m

    def forward_slopes(self, layers, a=None):
        """Noise-free s = Gamma (P phi - P_dm a) (simulation.hpp:164-199)."""
        x = _f64(layers)
        count = x.size // self.dims.n
        out = np.zeros(count * self.dims.S)
        self._chk(self._L.fewha_gpu_forward_slopes(self._h, _dp(x), _dp(None if a is None else _f64(a)), _dp(out), count))
        return out if count == 1 else out.reshape(count, self.dims.S)

    def wfs_operator(self, x=None, meas=None, rhs: bool = False):
        """The frame's fused per-WFS tile kernel (k_wfs) on its own:
        rhs=False: psi = Gamma^T C^-1 Gamma P x (x nodal layers [count, n]);
        rhs=True:  psi = Gamma^T C^-1 (meas + Gamma P_dm x) (x DM commands or None)."""
        d = self.dims
        if rhs:
            m = _f64(meas)
            count = m.size // d.S
            a = None if x is None else _f64(x, d.A * count)
        else:
            a = _f64(x)
            count = a.size // d.n
            m = None
        out = np.zeros(count * d.Nw)
        self._chk(self._L.fewha_gpu_wfs_operator(self._h, 1 if rhs else 0, _dp(a), _dp(m), _dp(out), count))
        return out if count == 1 else out.reshape(count, d.Nw)

    # -- CUDA-resident path -----------------------------------------------------------
    def enable_telemetry(self, on: bool = True):
        """StepTelemetry stage timings for every graph frame (opt-in, serialising)."""
        self._chk(self._L.fewha_gpu_enable_telemetry(self._h, 1 if on else 0))

    def last_telemetry(self) -> dict:
        """Reconstructor::last_telemetry(): step, stage1/2/3, pcg, fit, total (us), rho."""
        t = _Telemetry()
        self._chk(self._L.fewha_gpu_last_telemetry(self._h, C.byref(t)))
        out = {k: getattr(t, k) for k, _ in _Telemetry._fields_}
        out["valid"] = bool(out["valid"])
        out["rho"] = getattr(self, "last_rho", None)
        return out

    def last_launch_times(self):
        """[(kind, ms), ...] of the last graph frame (telemetry event nodes)."""
        ms = (C.c_float * 256)()
        kinds = (C.c_int * 256)()
        n = self._L.fewha_gpu_last_launch_times(self._h, ms, kinds, 256)
        if n < 0:
            self._chk(-n)
        return [(self.KERNEL_KINDS[kinds[i]], float(ms[i])) for i in range(n)]

    def shard(self, rank: int, world: int, nccl_id: bytes | None = None):
        """Own the WFS of shard rank/world.  nccl_id: multi-process
        NCCL exchange of the partial layer sums; None: in-process group member."""
        if nccl_id is not None and len(nccl_id) != 128:
            raise ArgumentError("nccl_id must be 128 bytes")
        self._chk(self._L.fewha_gpu_shard(self._h, rank, world, nccl_id))

    def shard_wfs(self) -> tuple[int, int]:
        b, e = C.c_int(), C.c_int()
        self._chk(self._L.fewha_gpu_shard_wfs(self._h, C.byref(b), C.byref(e)))
        return b.value, e.value

    def set_stream(self, stream_handle: int):
        self._chk(self._L.fewha_gpu_set_stream(self._h, C.c_void_p(stream_handle)))

    def device_buffers(self):
        b = _DevBufs()
        self._chk(self._L.fewha_gpu_device_buffers(self._h, C.byref(b)))
        return {k: getattr(b, k) for k, _ in _DevBufs._fields_}

    def load_slopes(self, slopes):
        """Stage host slopes [batch][S] into the resident slot (synchronous copy)."""
        s = _f64(slopes, self.dims.S * self.dims.batch)
        self._chk(self._L.fewha_gpu_load_slopes(self._h, s.ctypes.data_as(C.c_void_p), 0))
        self.sync()

    def load_slopes_device(self, d_ptr: int):
        """Stage device slopes [batch][S] fp64 into the resident slot (async)."""
        self._chk(self._L.fewha_gpu_load_slopes(self._h, C.c_void_p(d_ptr), 1))

    def step_device(self, d_slopes_ptr: int | None = None):
        self._chk(self._L.fewha_gpu_step_device(self._h, None if d_slopes_ptr is None else C.c_void_p(d_slopes_ptr)))

    def sync(self):
        self._chk(self._L.fewha_gpu_sync(self._h))

    def launches_per_step(self) -> int:
        return int(self._L.fewha_gpu_launches_per_step(self._h))

    def plan_info(self) -> dict:
        """The execution plan chosen for this handle's batch size (fewha_gpu_plan_info)."""
        p = _Plan()
        self._chk(self._L.fewha_gpu_plan_info(self._h, C.byref(p)))
        return {k: getattr(p, k) for k, _ in _Plan._fields_}

    def phase_stamps(self, enable_only=False):
        """Per-phase %globaltimer stamps of the cluster kernels of the last
        profile_step frame: array [launch][block][16] (ns; 0 = not stamped)."""
        if enable_only:
            self._chk(-min(0, self._L.fewha_gpu_phase_stamps(self._h, None, 0)))
            return None
        out = np.zeros(32 * 16384 * 16, np.uint64)
        n = self._L.fewha_gpu_phase_stamps(self._h, out.ctypes.data_as(C.c_void_p), out.size)
        if n < 0:
            self._chk(-n)
        return out.reshape(32, 16384, 16)

    KERNEL_KINDS = ("wfs_rhs", "adjoint", "fwd_rhs", "inv_pcg0", "inv_pcg", "wfs", "fwd_pcg", "inv_fit", "fit_control", "gather",
                    "fwd_rhs_inv0", "fwd_inv_pcg", "fwd_inv_fit")

    def profile_step(self):
        """One eager frame with events between launches: [(kind, ms), ...]."""
        ms = (C.c_float * 256)()
        kinds = (C.c_int * 256)()
        n = self._L.fewha_gpu_profile_step(self._h, ms, kinds, 256)
        if n < 0:
            self._chk(-n)
        return [(self.KERNEL_KINDS[kinds[i]], float(ms[i])) for i in range(n)]


def preset_info(path):
    """load_config + finalize_geometry on the host only (no device): returns
    (dims, layer_extent, dm_extent, masks).  Raises ConfigError like
    config_io.hpp:181."""
    L = lib()
    d = _Dims()
    p = os.fspath(path).encode()
    rc = L.fewha_gpu_preset_info(p, C.byref(d), None, None, None)
    if rc:
        raise _ERR.get(rc, FewhaError)(L.fewha_gpu_create_error().decode())
    ext, dext = np.zeros(d.n_layers), np.zeros(d.n_dms)
    masks = np.zeros(d.n_slopes // 2, np.uint8)
    L.fewha_gpu_preset_info(p, None, _dp(ext), _dp(dext), masks.ctypes.data_as(C.c_void_p))
    dims = Dims(d.n_coeff, d.n_slopes, d.n_act, d.n_wavefront, d.n_layers, d.n_wfs, d.n_dms, d.pcg_iters, 0, 0)
    return dims, ext, dext, masks
