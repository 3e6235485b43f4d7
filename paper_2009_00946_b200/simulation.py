"""Closed-loop simulation harness around the device reconstructor.

The reference's simulation layer (/root/reference/proj/include/fewha/
simulation.hpp) runs on the device (csrc/sim_kernels.cuh, driven by
csrc/engine.cu), so a closed loop moves no data between host and device per
frame; this module is the Python face of those C-ABI entry points:

  * ``gaussian_stream``     GaussianStream, simulation.hpp:40-58 (mt19937_64 + Box-Muller)
  * ``generate_atmosphere`` generate_atmosphere + truth_at_step, simulation.hpp:76-158
  * ``synthesize``          synthesize_measurements, simulation.hpp:164-212
  * ``evaluate_quality``    evaluate_quality, simulation.hpp:228-305
  * ``run_closed_loop``     run_closed_loop, simulation.hpp:321-345

Parity with the unmodified reference (oracle/_ref): tests/test_gpu_simulation.py.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

import paper_2009_00946_b200 as fg

MASK64 = (1 << 64) - 1


def splitmix64(x: int) -> int:
    """SplitMix64 finaliser (simulation.hpp:31-36): the per-frame noise seeds of
    run_bench / run_closed_loop are splitmix64(seed + k)."""
    x = (x + 0x9E3779B97F4A7C15) & MASK64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & MASK64
    return x ^ (x >> 31)


def _dp(a):
    return None if a is None else a.ctypes.data_as(C.POINTER(C.c_double))


def gaussian_stream(seed: int, count: int, device: int = 0) -> np.ndarray:
    """The first `count` (even) draws of GaussianStream(seed), generated on the device."""
    out = np.zeros(count)
    rc = fg.lib().fewha_gpu_sim_gauss(device, seed & MASK64, count, _dp(out))
    if rc:
        raise fg._ERR.get(rc, fg.FewhaError)(fg.lib().fewha_gpu_create_error().decode())
    return out


def generate_atmosphere(rec: "fg.Reconstructor", seed: int, step: int = 0) -> np.ndarray:
    """truth_at_step(generate_atmosphere(g, seed), g, step): nodal layers [n]."""
    out = np.zeros(rec.dims.n)
    rec._chk(rec._L.fewha_gpu_sim_atmosphere(rec._h, seed & MASK64, step, _dp(out)))
    return out


def synthesize(rec: "fg.Reconstructor", layers, correction, noise_seed: int) -> np.ndarray:
    """synthesize_measurements(layers, correction or None, g, noise_seed)."""
    lay = np.ascontiguousarray(layers, np.float64).ravel()
    a = None if correction is None else np.ascontiguousarray(correction, np.float64).ravel()
    out = np.zeros(rec.dims.S)
    rec._chk(rec._L.fewha_gpu_sim_synthesize(rec._h, _dp(lay), _dp(a), noise_seed & MASK64, _dp(out)))
    return out


@dataclass
class QualityRecord:
    step: int = 0
    rms_per_dir: np.ndarray = field(default_factory=lambda: np.zeros(0))
    field_rms: float = 0.0
    layer_rel_err: float = 0.0  # NaN without the reference's L = M pairing
    rho: np.ndarray = field(default_factory=lambda: np.zeros(0))

    @staticmethod
    def of(rec_row, step=0, rho=None):
        return QualityRecord(step, np.array(rec_row[2:]), float(rec_row[0]), float(rec_row[1]),
                             np.zeros(0) if rho is None else np.array(rho))


def evaluate_quality(rec: "fg.Reconstructor", layers, correction) -> QualityRecord:
    """evaluate_quality(truth layers, DM correction, g) on the device."""
    lay = np.ascontiguousarray(layers, np.float64).ravel()
    a = np.ascontiguousarray(correction, np.float64).ravel()
    n = rec._L.fewha_gpu_sim_quality_size(rec._h)
    if n < 0:
        rec._chk(-n)
    out = np.zeros(n)
    rec._chk(rec._L.fewha_gpu_sim_quality(rec._h, _dp(lay), _dp(a), _dp(out)))
    return QualityRecord.of(out)


@dataclass
class LoopResult:
    records: list
    uncorrected_field_rms: float
    final_field_rms: float


def run_closed_loop(preset, n_steps: int, atmosphere_seed: int = 1, noise_seed: int = 2, precision: int = 64,
                    device: int = 0, rec: "fg.Reconstructor | None" = None) -> LoopResult:
    """run_closed_loop (simulation.hpp:321-345) with every frame on the device:
    at step k the slopes and the quality see a^(k-1), the frame produces
    a^(k+1); one device-to-host copy of the records at the end."""
    if n_steps < 1:
        raise fg.ArgumentError("run_closed_loop: n_steps must be >= 1")
    if rec is None:
        rec = fg.Reconstructor(preset, precision=precision, device=device)
    n = rec._L.fewha_gpu_sim_quality_size(rec._h)
    if n < 0:
        rec._chk(-n)
    recs = np.zeros((n_steps, n))
    rho = np.zeros((n_steps, rec.dims.iters))
    uf = np.zeros(2)
    rec._chk(rec._L.fewha_gpu_run_closed_loop(rec._h, n_steps, atmosphere_seed & MASK64, noise_seed & MASK64,
                                              _dp(recs), _dp(rho), _dp(uf)))
    records = [QualityRecord.of(recs[k], k, rho[k]) for k in range(n_steps)]
    return LoopResult(records, float(uf[0]), float(uf[1]))
