"""Closed-loop simulation harness around the device reconstructor.

A restatement of the reference's simulation layer
(/root/reference/proj/include/fewha/simulation.hpp) that drives the sm_100a
frame (`fewha_gpu_step`) instead of the CPU solver:

  * ``GaussianStream``       simulation.hpp:40-58   mt19937_64 bits -> Box-Muller pairs
  * ``generate_atmosphere``  simulation.hpp:76-127  von Karman screens by spectral sampling
  * ``truth_at_step``        simulation.hpp:131-158 periodic frozen-flow translation
  * ``synthesize``           simulation.hpp:164-212 the device forward model
                             Gamma (P phi - P_dm a) (fewha_gpu_forward_slopes) plus the
                             reference's noise stream on the active subapertures
  * ``evaluate_quality``     simulation.hpp:228-305 piston-removed residual RMS per probe
                             direction, field RMS, layer reconstruction error
  * ``run_closed_loop``      simulation.hpp:321-345 two-step-delay loop

The random streams, the screen synthesis and the quality metrics are host
numpy (they feed and observe the path, they are not on it); the slopes'
noise-free part and every reconstruction run on the GPU.  Parity with the
reference's own run_closed_loop: tests/test_gpu_simulation.py.
"""
from __future__ import annotations

import json
import math
import os
from dataclasses import dataclass, field

import numpy as np

import paper_2009_00946_b200 as fg

MASK64 = (1 << 64) - 1
ARCSEC = math.pi / (180.0 * 3600.0)  # kArcsecToRad


def splitmix64(x: int) -> int:
    """SplitMix64 finaliser (simulation.hpp:31-36), on Python ints mod 2^64."""
    x = (x + 0x9E3779B97F4A7C15) & MASK64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & MASK64
    return x ^ (x >> 31)


class MT19937_64:
    """std::mt19937_64 (Matsumoto-Nishimura 64-bit Mersenne Twister), block-vectorised.

    The twist of the 312-word state splits into two data-parallel halves: words
    [0, 156) read only old words, words [156, 311) read the new words 156 back,
    and word 311 reads the new word 0."""

    N, M = 312, 156
    A = np.uint64(0xB5026F5AA96619E9)
    UM, LM = np.uint64(0xFFFFFFFF80000000), np.uint64(0x7FFFFFFF)

    def __init__(self, seed: int):
        mt = [seed & MASK64]
        for i in range(1, self.N):
            prev = mt[-1]
            mt.append((6364136223846793005 * (prev ^ (prev >> 62)) + i) & MASK64)
        self.mt = np.array(mt, dtype=np.uint64)
        self.buf = np.empty(0, dtype=np.uint64)

    def _twist(self):
        mt, M, one = self.mt, self.M, np.uint64(1)

        def mix(cur, nxt, far):
            x = (cur & self.UM) | (nxt & self.LM)
            xa = x >> one
            return far ^ np.where((x & one) != 0, xa ^ self.A, xa)

        new = np.empty_like(mt)
        new[:M] = mix(mt[:M], mt[1:M + 1], mt[M:])
        new[M:self.N - 1] = mix(mt[M:self.N - 1], mt[M + 1:], new[:self.N - 1 - M])
        new[self.N - 1:] = mix(mt[self.N - 1:], new[:1], new[M - 1:M])
        self.mt = new
        y = new.copy()
        y ^= (y >> np.uint64(29)) & np.uint64(0x5555555555555555)
        y ^= (y << np.uint64(17)) & np.uint64(0x71D67FFFEDA60000)
        y ^= (y << np.uint64(37)) & np.uint64(0xFFF7EEE000000000)
        y ^= y >> np.uint64(43)
        return y

    def draws(self, count: int) -> np.ndarray:
        out = [self.buf]
        have = self.buf.size
        while have < count:
            blk = self._twist()
            out.append(blk)
            have += blk.size
        allv = np.concatenate(out)
        self.buf = allv[count:]
        return allv[:count]


class GaussianStream:
    """Deterministic standard normals (simulation.hpp:40-58): per pair, u1 from
    (bits >> 11) + 1 (so in (0, 1]), u2 from the next draw's bits >> 11, both
    scaled by 2^-53; returns m cos(a) then m sin(a), m = sqrt(-2 ln u1),
    a = 2 pi u2."""

    def __init__(self, seed: int):
        self.rng = MT19937_64(seed)
        self.cache = None

    def take(self, count: int) -> np.ndarray:
        out = np.empty(count)
        k = 0
        if self.cache is not None and count > 0:
            out[0] = self.cache
            self.cache = None
            k = 1
        pairs = (count - k + 1) // 2
        if pairs > 0:
            bits = self.rng.draws(2 * pairs)
            u1 = ((bits[0::2] >> np.uint64(11)).astype(np.float64) + 1.0) * 2.0 ** -53
            u2 = (bits[1::2] >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
            m = np.sqrt(-2.0 * np.log(u1))
            a = 2.0 * math.pi * u2
            vals = np.empty(2 * pairs)
            vals[0::2] = m * np.cos(a)
            vals[1::2] = m * np.sin(a)
            need = count - k
            out[k:] = vals[:need]
            if need < vals.size:
                self.cache = vals[need]
        return out


@dataclass
class SimGeometry:
    """The preset fields the simulation reads, with the reference's defaults
    (config_io.hpp:71-175) and its derived extents/masks (finalize_geometry)."""

    diameter: float
    r_out: float
    r_in: float
    layers: list            # (side, height, relative_strength, extent)
    dms: list               # (n_act, height, extent)
    stars: list             # (kind, theta_x, theta_y, height)
    wfs: list               # (n_subap, noise_variance)
    masks: list             # active masks per WFS (n_s x n_s uint8)
    outer_scale: float
    truth_strength: float
    noise: bool
    wind: list              # per layer (vx, vy) m/step, or []
    n_per_side: int
    half_width: float
    paired: bool            # L == M identity pairing (layer_rel_err defined)

    @staticmethod
    def load(preset) -> "SimGeometry":
        j = json.load(open(preset)) if isinstance(preset, (str, os.PathLike)) else preset
        path = preset
        if not isinstance(preset, (str, os.PathLike)):
            import tempfile
            fd, path = tempfile.mkstemp(suffix=".json")
            with os.fdopen(fd, "w") as f:
                json.dump(j, f)
        try:
            dims, ext, dext, masks = fg.preset_info(path)
        finally:
            if path is not preset:
                os.unlink(path)
        tel = j["telescope"]
        D = float(tel["diameter"])
        frac = float(tel.get("obstruction_fraction", 0.0))
        sem = tel.get("obstruction_semantics", "area")
        f = math.sqrt(frac) if sem == "area" else frac

        def direction(js, key):
            if key + "_rad" in js:
                return tuple(float(v) for v in js[key + "_rad"])
            return tuple(float(v) * ARCSEC for v in js[key + "_arcsec"])

        stars = []
        for s in j["guide_stars"]:
            tx, ty = direction(s, "direction")
            lgs = s["kind"] == "lgs"
            stars.append(("lgs" if lgs else "ngs", tx, ty, float(s["height"]) if lgs else math.inf))
        layers = [(1 << int(l["grid_order"]), float(l["height"]), float(l["relative_strength"]), float(e))
                  for l, e in zip(j["layers"], ext)]
        dms = [(int(d["n_act"]), float(d["conjugation_height"]), float(e)) for d, e in zip(j["dms"], dext)]
        wfs = [(int(w["n_subap"]), float(w["noise_variance"])) for w in j["wfs"]]
        mk, off = [], 0
        for ns, _ in wfs:
            mk.append(masks[off:off + ns * ns].reshape(ns, ns))
            off += ns * ns
        ev = j.get("evaluation", {})
        if "half_width_rad" in ev:
            hw = float(ev["half_width_rad"])
        else:
            hw = float(ev.get("half_width_arcsec", 60.0)) * ARCSEC
        sim = j.get("simulation", {})
        wind = [tuple(float(x) for x in v) for v in sim.get("wind_m_per_step", [])]
        return SimGeometry(D, D / 2.0, f * D / 2.0, layers, dms, stars, wfs, mk,
                           float(j["solver"].get("outer_scale", 25.0)), float(sim.get("truth_strength", 1.0)),
                           bool(sim.get("noise", True)), wind, int(ev.get("n_per_side", 5)), hw,
                           j.get("fitting", "identity") != "projection" and len(layers) == len(dms))

    def directions(self):
        """EvaluationConfig::directions (geometry.hpp:122-133): row-major square grid."""
        n, hw = self.n_per_side, self.half_width
        out = []
        for i in range(n):
            for jj in range(n):
                fy = 0.0 if n == 1 else -1.0 + 2.0 * i / (n - 1)
                fx = 0.0 if n == 1 else -1.0 + 2.0 * jj / (n - 1)
                out.append((fx * hw, fy * hw))
        return out


# ---- screens ------------------------------------------------------------------

def generate_atmosphere(geo: SimGeometry, seed: int) -> list[np.ndarray]:
    """Von Karman screens (simulation.hpp:76-127): per layer, complex white noise
    from GaussianStream(splitmix64(seed ^ (0x51a9e4c7 + l))) drawn row-major as
    (re, im) pairs, shaped by (k^2 + k0^2)^(-11/12) on the screen's periodic
    grid (period = spacing * n), DC zeroed, inverse 2-D FFT, real part, mean
    removed, variance scaled to relative_strength * truth_strength."""
    k0 = 2.0 * math.pi / geo.outer_scale
    out = []
    for l, (n, _h, strength, extent) in enumerate(geo.layers):
        period = extent / (n - 1) * n
        g = GaussianStream(splitmix64(seed ^ ((0x51A9E4C7 + l) & MASK64)))
        z = g.take(2 * n * n)
        # wavenumber index wi = ki for ki <= n/2, else ki - n (simulation.hpp:89-92)
        w = np.where(np.arange(n) <= n // 2, np.arange(n), np.arange(n) - n).astype(np.float64)
        kx = 2.0 * math.pi * w[None, :] / period
        ky = 2.0 * math.pi * w[:, None] / period
        amp = (kx * kx + ky * ky + k0 * k0) ** (-11.0 / 12.0)
        spec = (z[0::2] + 1j * z[1::2]).reshape(n, n) * amp
        spec[0, 0] = 0.0
        scr = np.real(np.fft.ifft2(spec))
        scr = scr - scr.mean()
        var = float(np.mean(scr * scr))
        target = strength * geo.truth_strength
        out.append(scr * (math.sqrt(target / var) if var > 0.0 else 0.0))
    return out


def truth_at_step(geo: SimGeometry, truth: list[np.ndarray], step: int) -> list[np.ndarray]:
    """Periodic frozen flow (simulation.hpp:131-158): screen l translated by
    wind_l * step / spacing nodes with periodic bilinear interpolation."""
    if not geo.wind or step == 0:
        return truth
    out = []
    for (n, _h, _s, extent), base, (vx, vy) in zip(geo.layers, truth, geo.wind):
        sp = extent / (n - 1)
        si, sj = vy * step / sp, vx * step / sp
        ti = np.mod(np.arange(n) + si, float(n))
        tj = np.mod(np.arange(n) + sj, float(n))
        ti = np.where(ti < 0, ti + n, ti)
        tj = np.where(tj < 0, tj + n, tj)
        i0 = ti.astype(np.int64) % n
        j0 = tj.astype(np.int64) % n
        i1, j1 = (i0 + 1) % n, (j0 + 1) % n
        fi = (ti - np.floor(ti))[:, None]
        fj = (tj - np.floor(tj))[None, :]
        b = base
        out.append((1 - fi) * ((1 - fj) * b[np.ix_(i0, j0)] + fj * b[np.ix_(i0, j1)]) +
                   fi * ((1 - fj) * b[np.ix_(i1, j0)] + fj * b[np.ix_(i1, j1)]))
    return out


# ---- measurements ---------------------------------------------------------------

def synthesize(rec: "fg.Reconstructor", geo: SimGeometry, layers: list[np.ndarray], correction,
               noise_seed: int) -> np.ndarray:
    """synthesize_measurements (simulation.hpp:164-212): the noise-free slopes
    Gamma (P phi - P_dm a) from the device forward model, then, when the preset's
    simulation noise is on, sigma_w * N(0,1) on sx then sy of every active
    subaperture, WFS by WFS in row-major order, from one
    GaussianStream(splitmix64(noise_seed ^ 0x6e0f7a3d))."""
    s = rec.forward_slopes(np.concatenate([l.ravel() for l in layers]),
                           None if correction is None else np.asarray(correction, np.float64))
    s = np.array(s, dtype=np.float64).ravel()
    if geo.noise:
        g = GaussianStream(splitmix64(noise_seed ^ 0x6E0F7A3D))
        off = 0
        for (ns, var), mask in zip(geo.wfs, geo.masks):
            act = np.flatnonzero(mask.ravel())
            z = g.take(2 * act.size)
            sig = math.sqrt(var)
            s[off + act] += sig * z[0::2]
            s[off + ns * ns + act] += sig * z[1::2]
            off += 2 * ns * ns
    return s


# ---- quality --------------------------------------------------------------------

def _bilinear(v: np.ndarray, extent: float, px: np.ndarray, py: np.ndarray) -> np.ndarray:
    """bilinear_sample (operators.hpp:108-127), vectorised; off-grid points raise."""
    n = v.shape[0]
    sp = extent / (n - 1)
    u = (px + extent / 2.0) / sp
    t = (py + extent / 2.0) / sp
    eps = 1e-9
    if np.any(u < -eps) or np.any(u > n - 1 + eps) or np.any(t < -eps) or np.any(t > n - 1 + eps):
        raise fg.FewhaError("propagation: evaluation point outside layer grid")
    j0 = np.minimum(np.floor(u).astype(np.int64), n - 2)
    i0 = np.minimum(np.floor(t).astype(np.int64), n - 2)
    fx, fy = u - j0, t - i0
    i0, j0 = np.maximum(i0, 0), np.maximum(j0, 0)
    return ((1 - fy) * (1 - fx) * v[i0, j0] + (1 - fy) * fx * v[i0, j0 + 1] + fy * (1 - fx) * v[i0 + 1, j0] +
            fy * fx * v[i0 + 1, j0 + 1])


def _split_dm(geo: SimGeometry, a) -> list[np.ndarray]:
    a = np.asarray(a, np.float64).ravel()
    out, off = [], 0
    for n, _h, _e in geo.dms:
        out.append(a[off:off + n * n].reshape(n, n))
        off += n * n
    return out


@dataclass
class QualityRecord:
    step: int = 0
    rms_per_dir: np.ndarray = field(default_factory=lambda: np.zeros(0))
    field_rms: float = 0.0
    layer_rel_err: float = 0.0
    rho: np.ndarray = field(default_factory=lambda: np.zeros(0))


def evaluate_quality(geo: SimGeometry, layers: list[np.ndarray], correction) -> QualityRecord:
    """evaluate_quality (simulation.hpp:228-305): for every probe direction the
    truth minus the DM correction propagated to the annular-pupil nodes of the
    finest WFS grid, piston removed, RMS; the field RMS is their quadratic mean;
    layer_rel_err compares the DM shapes resampled on the layer grids with the
    truth (mean-removed; L = M identity pairing only, else NaN)."""
    n = max(ns for ns, _ in geo.wfs) + 1
    d = geo.diameter / (n - 1)
    xs = -geo.r_out + np.arange(n) * d
    X, Y = np.meshgrid(xs, xs)  # Y[i, j] = -r_out + i d
    r2 = X * X + Y * Y
    sel = (r2 <= geo.r_out ** 2 * (1.0 + 1e-12)) & (r2 >= geo.r_in ** 2 * (1.0 - 1e-12))
    px, py = X[sel], Y[sel]  # row-major node order
    dms = _split_dm(geo, correction)
    rec = QualityRecord()
    rms, sum_sq = [], 0.0
    for tx, ty in geo.directions():
        res = np.zeros(px.size)
        for (nl, h, _s, ext), lay in zip(geo.layers, layers):
            res += _bilinear(lay, ext, px + tx * h, py + ty * h)
        for (na, h, ext), dm in zip(geo.dms, dms):
            res -= _bilinear(dm, ext, px + tx * h, py + ty * h)
        mean = float(np.sum(res)) / res.size
        var = float(np.sum((res - mean) ** 2)) / res.size
        rms.append(math.sqrt(var))
        sum_sq += var
    rec.rms_per_dir = np.array(rms)
    rec.field_rms = math.sqrt(sum_sq / len(rms))
    if geo.paired:
        num = den = 0.0
        for (nl, _h, _s, ext), lt, dm in zip(geo.layers, layers, dms):
            c = -ext / 2.0 + np.arange(nl) * (ext / (nl - 1))
            CX, CY = np.meshgrid(c, c)
            up = _bilinear(dm, ext, CX.ravel(), CY.ravel()).reshape(nl, nl)
            diff = (up - up.mean()) - (lt - lt.mean())
            num += float(np.sum(diff * diff))
            den += float(np.sum((lt - lt.mean()) ** 2))
        rec.layer_rel_err = math.sqrt(num / den) if den > 0.0 else 0.0
    else:
        rec.layer_rel_err = float("nan")
    return rec


# ---- the loop --------------------------------------------------------------------

@dataclass
class LoopResult:
    records: list
    uncorrected_field_rms: float
    final_field_rms: float


def run_closed_loop(preset, n_steps: int, atmosphere_seed: int = 1, noise_seed: int = 2, precision: int = 64,
                    device: int = 0, rec: "fg.Reconstructor | None" = None) -> LoopResult:
    """run_closed_loop (simulation.hpp:321-345) on the device reconstructor: at
    step k the slopes and the quality see a^(k-1) (the state's a_prev2), the
    frame produces a^(k+1); slopes synthesised with noise seed
    splitmix64(noise_seed + k)."""
    if n_steps < 1:
        raise fg.ArgumentError("run_closed_loop: n_steps must be >= 1")
    geo = SimGeometry.load(preset)
    truth = generate_atmosphere(geo, atmosphere_seed)
    if rec is None:
        rec = fg.Reconstructor(preset, precision=precision, device=device)
    rec.build_preconditioner()
    A = sum(n * n for n, _h, _e in geo.dms)
    a_prev2, a_prev = np.zeros(A), np.zeros(A)
    records, layers_k = [], truth
    for k in range(n_steps):
        layers_k = truth_at_step(geo, truth, k)
        meas = synthesize(rec, geo, layers_k, a_prev2, splitmix64((noise_seed + k) & MASK64))
        q = evaluate_quality(geo, layers_k, a_prev2)
        q.step = k
        a_new = np.array(rec.step(meas, want_coeffs=False), dtype=np.float64)
        q.rho = np.array(rec.last_rho)
        records.append(q)
        a_prev2, a_prev = a_prev, a_new  # ReconstructorState rotation (reconstructor.hpp:349-350)
    unc = evaluate_quality(geo, layers_k, np.zeros(A)).field_rms
    return LoopResult(records, unc, records[-1].field_rms)
