#!/usr/bin/env python
"""Benchmark of the FEWHA reconstruction frame (Reconstructor::step) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--precision 64|32] [--preset presets/elt_mcao84_3dm.json]

Workload (BASELINE.json metric "per-frame reconstruction latency p50/p99 (ms)
and recon/sec vs memory roofline", config 3): ELT MCAO-84 -- 39 m, 6 LGS 84x84
+ 3 NGS, 9 layers of 128^2 (J=7), 3 DMs (81^2, 48^2, 54^2), closed loop, 4
warm-started PCG iterations, fp64 (presets/elt_mcao84_3dm.json; the 3-DM
fitting is the projection extension).  One step = one frame of one
instance.  The reference supports only L = M, so its CPU arm runs the L = M
shadow of the same preset (same layers, WFS and PCG; 9 identity-fitted DMs).

  value      reconstructions/s over all ranks, slopes resident in HBM, timed with
             CUDA events around each frame's graph launch; L2 flushed (256 MiB
             write) before every timed frame.  `latency`: a separate >= 1000-frame
             sample of the same (p50/p99 need it whatever --steps is).
  e2e        the same metric through the C-ABI fewha_gpu_step with HOST buffers
             (H2D of the frame's slopes + a^(1), rho and status back inside the
             timed region): a registered slope ring (headline) and, beside it,
             ordinary pageable arrays (the reference's calling convention).
  roofline   the dominant kernel FUNCTION (largest share of the frame, its launch
             kinds summed), timed by event-record nodes between the launches of the
             captured frame graph: algorithmic bytes per launch / its mean launch
             time; `traffic` = its ncu DRAM bytes per launch (profiles/dram_traffic.json).
  cpu_baseline  the reference solver (oracle/_ref, compiled from the unmodified
             reference) timed on this host's cores on a bounded frame sample, with
             the CPU model.
  shard      (N > 1) the per-WFS split of one instance's frame over the N ranks
             (the north star's partition), next to the replicas value.

--impl reference runs the reference CPU solver alone (rank 0), with every
host thread, on the same config and slope stream.
N > 1: one process per GPU, independent instances per rank (replicas,
"scaling": "weak"); the path has no exchange step in this mode.
--shard (N > 1): per-WFS sharding of ONE instance's frame: rank r
owns a contiguous WFS range, the partial adjoint layer sums are all-reduced
through NCCL inside the frame graph; value = frames/s of that one instance
("scaling": "strong").
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "per-frame reconstruction latency p50/p99 (ms) and recon/sec vs memory roofline"
UNIT = "recon/s"
DEFAULT_PRESET = os.path.join(ROOT, "presets", "elt_mcao84_3dm.json")
L2_FLUSH_BYTES = 256 << 20


def load_json(path):
    with open(path) as f:
        return json.load(f)


def preset_dims(preset):
    j = load_json(preset)
    ns = [w["n_subap"] for w in j["wfs"]]
    n = sum((1 << l["grid_order"]) ** 2 for l in j["layers"])
    S = sum(2 * k * k for k in ns)
    Nw = sum((k + 1) ** 2 for k in ns)
    A = sum(d["n_act"] ** 2 for d in j["dms"])
    return dict(n=n, S=S, Nw=Nw, A=A, L=len(j["layers"]), W=len(ns), M=len(j["dms"]),
                iters=j["solver"]["pcg_max_iter"], closed=j["loop"]["mode"] == "closed")


def frame_bytes(d, b):
    """Fused-minimum algorithmic traffic of one frame (SURVEY.md 8d / BASELINE.md 4)."""
    n, S, Nw, A, it = d["n"], d["S"], d["Nw"], d["A"], d["iters"]
    A_cl = A if d["closed"] else 0
    return b * (it * (13 * n + 2 * Nw) + (4 * n + 2 * Nw + A_cl) + (n + 3 * A)) + 8 * S


def kernel_bytes(kind, d, b):
    """Algorithmic bytes of one launch of each kernel kind (one instance):
    every array the kernel must read or write crosses memory once."""
    n, S, Nw, A = d["n"], d["S"], d["Nw"], d["A"]
    return {
        "wfs_rhs": 8 * S + b * (A + Nw),          # slopes (fp64) + a_prev2 -> psi
        "adjoint": b * (Nw + n),                  # psi -> y (legacy kind id)
        "gather": b * (Nw + n),                   # psi -> y (k_gather)
        "fwd_rhs": b * (3 * n + 2 * n),           # y, r, b -> r, b
        "inv_pcg0": b * (2 * n + n),              # r, J -> phi
        "inv_pcg": b * (6 * n + 4 * n + n),       # r, J, p, q, c, Mz -> p, q, c, r, phi
        "wfs": b * (n + Nw),                      # phi -> psi
        "fwd_pcg": b * (3 * n + n),               # y, r, J -> Mz
        "inv_fit": b * (6 * n + 4 * n + n),       # last update + c -> phi
        "fit_control": b * (n + 5 * A),           # phi, a_prev, a_prev2 -> a_prev2, a_prev, a_out
        # fused forward + inverse (k_fwd_inv_cluster): Mz / the RHS pass no longer cross memory
        "fwd_rhs_inv0": b * (4 * n + 3 * n),      # y, r, b, J -> r, b, phi
        "fwd_inv_pcg": b * (6 * n + 5 * n),       # y, r, J, p, q, c -> p, q, c, r, phi
        "fwd_inv_fit": b * (6 * n + 5 * n),       # y, r, J, p, q, c -> p, q, c, r, phi
    }[kind]


def synthetic_layers(preset, seed):
    """Von Karman layer screens (FFT-shaped complex noise, simulation.hpp:76-127
    spectrum (k^2 + k0^2)^(-11/12)), strength-scaled; nodal [n]."""
    j = load_json(preset)
    L0 = j["solver"].get("outer_scale", 25.0)
    rng = np.random.default_rng(seed)
    out = []
    for lay in j["layers"]:
        n = 1 << lay["grid_order"]
        ext = 1.0  # physical scale irrelevant for the synthetic stream shape
        f = np.fft.fftfreq(n, d=ext / n)
        kk = (2 * np.pi) ** 2 * (f[:, None] ** 2 + f[None, :] ** 2) + (2 * np.pi / L0) ** 2
        amp = kk ** (-11.0 / 12.0)
        amp[0, 0] = 0.0
        scr = np.real(np.fft.ifft2((rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) * amp))
        scr -= scr.mean()
        scr *= math.sqrt(lay["relative_strength"]) / max(scr.std(), 1e-30)
        out.append(scr.ravel())
    return np.concatenate(out)


def slope_stream(rec, preset, frames, seed):
    """Noisy slopes of frozen-flow-free random atmospheres: s = Gamma P phi + n
    (forward model on the GPU through the library, noise sigma_w per WFS)."""
    j = load_json(preset)
    layers = np.stack([synthetic_layers(preset, seed * 1000 + k) for k in range(frames)])
    s = rec.forward_slopes(layers).reshape(frames, -1)
    rng = np.random.default_rng(seed)
    sig = np.repeat([math.sqrt(w["noise_variance"]) for w in j["wfs"]], [2 * w["n_subap"] ** 2 for w in j["wfs"]])
    return np.ascontiguousarray(s + sig[None, :] * rng.standard_normal(s.shape))


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        time.sleep(0.25)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def peaks():
    try:
        p = load_json(os.path.join(ROOT, "MEASURED_PEAKS.json"))
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def reference_preset(preset):
    """The reference accepts only L = M: for a projection-fitting preset return
    its L = M shadow (same layers, WFS, solver; one DM per layer)."""
    j = load_json(preset)
    if j.get("fitting", "identity") != "projection":
        return preset
    j.pop("fitting", None)
    j["dms"] = [{"n_act": 1 << l["grid_order"], "conjugation_height": l["height"]} for l in j["layers"]]
    path = os.path.join("/tmp", "fewha_ref_shadow_" + os.path.basename(preset))
    with open(path, "w") as f:
        json.dump(j, f)
    return path


def cpu_reference_time(preset, stream, frames, threads):
    """Reference solver (oracle/_ref) on this host: per-frame wall times (us)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import RefOracle  # noqa: E402
    r = RefOracle(reference_preset(preset), threads=threads)
    r.build_preconditioner()
    r.time_steps(stream[:2], 2)  # warm-up frames
    us = r.time_steps(stream, frames)
    return us, r.threads


def host_slope_ring(frames, torch):
    """The e2e input ring as an AO real-time host would hold it: the frames in
    2 MB transparent-huge-page memory registered with CUDA (one DMA translation per
    2 MB instead of per 4 KB page -- rotating 4 KB-page buffers measured 5-45 us
    slower per call on these hosts, tools/e2e_break.py); falls back to
    torch.pin_memory()."""
    import mmap
    try:
        from cuda.bindings import runtime as rt
        hp = 2 << 20
        nbytes = frames.nbytes
        mm = mmap.mmap(-1, nbytes + 2 * hp, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
        base = np.frombuffer(mm, dtype=np.uint8)
        off = (-base.ctypes.data) % hp
        mm.madvise(mmap.MADV_HUGEPAGE, off, nbytes + hp)
        ring = base[off:off + nbytes].view(np.float64).reshape(frames.shape)
        ring[:] = frames
        if rt.cudaHostRegister(ring.ctypes.data, nbytes, rt.cudaHostRegisterDefault)[0] != rt.cudaError_t.cudaSuccess:
            raise RuntimeError("cudaHostRegister failed")
        host_slope_ring.keep = (mm, ring)  # lives for the process
        return torch.from_numpy(ring), "slope ring in 2 MB THP memory registered with cudaHostRegister"
    except Exception as e:  # noqa: BLE001
        return torch.from_numpy(frames).pin_memory(), f"slope ring in torch pinned memory ({type(e).__name__})"


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import RefOracle  # noqa: E402
    if not RefOracle.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built (needs /root/reference at build time)"}))
        return 0
    d = preset_dims(args.preset)
    threads = os.cpu_count() or 1
    rng = np.random.default_rng(7)
    # reference-side slope stream: the reference's own synthesis (bench.hpp:144-154 pattern)
    r = RefOracle(reference_preset(args.preset), threads=threads)
    stream = np.stack([r.synthesize(1, k) for k in range(4)])
    r.build_preconditioner()
    r.time_steps(stream, max(args.warmup, 1))
    us = r.time_steps(stream, args.steps)
    ms = us / 1000.0
    val = 1000.0 / float(np.mean(ms))
    line = {
        "impl": "reference", "metric": METRIC, "value": round(val, 3), "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(float(np.mean(ms)), 4),
        "p50_ms": round(float(np.percentile(ms, 50)), 4), "p99_ms": round(float(np.percentile(ms, 99)), 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "ELT MCAO-84 single-instance frame, reference CPU solver "
                               "(L=M shadow of the 3-DM preset: the reference supports only L=M)",
                   "preset": os.path.relpath(args.preset, ROOT), "threads": r.threads},
        "cpu_baseline": {"value": round(val, 3), "unit": UNIT, "cores": r.threads, "kind": "reference",
                         "cpu_model": cpu_model(), "nproc": os.cpu_count(),
                         "sample": f"{args.steps} frames of Reconstructor::step after {max(args.warmup,1)} warm-up, "
                                   f"{r.threads} pool threads on {os.cpu_count()} host cpus"},
        "e2e": {"value": round(val, 3), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# kernel kind (fewha_gpu_profile_step / last_launch_times) -> kernel function
FUNC = {"wfs_rhs": "k_wfs", "wfs": "k_wfs", "gather": "k_gather", "adjoint": "k_gather",
        "fwd_rhs": "k_fwd_cluster", "fwd_pcg": "k_fwd_cluster",
        "inv_pcg0": "k_inv_cluster", "inv_pcg": "k_inv_cluster", "inv_fit": "k_inv_cluster",
        "fit_control": "k_fit_control",
        "fwd_rhs_inv0": "k_fwd_inv_cluster", "fwd_inv_pcg": "k_fwd_inv_cluster", "fwd_inv_fit": "k_fwd_inv_cluster"}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def graph_function_profile(rec, frames, before, d, b, batch=1):
    """Per-kernel-function device times inside the captured frame graph: the
    telemetry event-record nodes between launches (fewha_gpu_last_launch_times).
    before(f) runs ahead of frame f (slope load, L2 flush).  Returns
    {function: {launches, ms_per_frame, bytes_per_frame, ...}} and the frame ms."""
    rec.enable_telemetry(True)
    plan = rec.plan_info()
    whole = plan.get("whole_layer", 0) >= 1  # batched plans: whole-layer transform kernels (2: fwd+inv fused)
    gdirect = plan.get("gather_direct", 0) == 1  # the direct gather (k_gather_direct)
    acc, frame_ms = {}, []
    for f in range(frames + 2):
        before(f)
        rec.step_device(None)
        lt = rec.last_launch_times()
        if f < 2:
            continue  # the first telemetry frames re-capture the graph
        frame_ms.append(sum(t for _, t in lt))
        for kind, t in lt:
            fn = FUNC[kind]
            if whole and fn in ("k_fwd_cluster", "k_inv_cluster", "k_fwd_inv_cluster"):
                fn = fn.replace("_cluster", "_layer")
            if gdirect and fn == "k_gather":
                fn = "k_gather_direct"
            e = acc.setdefault(fn, {"launches": 0, "ms": 0.0, "bytes": 0})
            e["launches"] += 1
            e["ms"] += t
            e["bytes"] += kernel_bytes(kind, d, b) * batch
    rec.enable_telemetry(False)
    rec.sync()
    tot = sum(frame_ms)
    out = {}
    for fn, e in acc.items():
        out[fn] = {"launches_per_frame": e["launches"] // frames, "ms_per_frame": e["ms"] / frames,
                   "launch_ms": e["ms"] / e["launches"], "bytes_per_launch": e["bytes"] / e["launches"],
                   "share": e["ms"] / tot, "achieved_gbs": e["bytes"] / (e["ms"] / 1000.0) / 1e9}
    return out, float(np.mean(frame_ms))


def roofline_object(prof, peak, peak_kind, traffic_key, note):
    dom = max(prof, key=lambda k: prof[k]["share"])
    e = prof[dom]
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "dram_traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = load_json(tpath).get(traffic_key, {}).get(dom)
        except Exception:
            traffic = None
    return {"bound": "hbm", "kernel": dom, "achieved": round(e["achieved_gbs"], 2), "peak": peak, "unit": "GB/s",
            "frac": round(e["achieved_gbs"] / peak, 4), "traffic": traffic,
            "bytes_per_launch": int(e["bytes_per_launch"]), "launch_ms": round(e["launch_ms"], 5),
            "launches_per_frame": e["launches_per_frame"], "share_of_frame": round(e["share"], 3),
            "peak_source": peak_kind, "timing": note,
            "functions": {k: {"share": round(v["share"], 3), "launch_ms": round(v["launch_ms"], 5),
                              "frac": round(v["achieved_gbs"] / peak, 4)}
                          for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["share"])}}


def e2e_loop(rec, lib, slopes_ptrs, a_ptr, r_ptr, frames, warm, flush, dev, torch):
    """fewha_gpu_step through the C-ABI with host buffers: per-call wall ms."""
    import ctypes as C
    import gc
    nr = (C.c_int * 1)()
    step_fn, h = lib.fewha_gpu_step, rec._h
    gc_was = gc.isenabled()
    gc.disable()  # real-time hygiene of an AO host loop
    out = []
    try:
        for k in range(warm + frames):
            sp = slopes_ptrs[k % len(slopes_ptrs)]
            flush.zero_()
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            code = step_fn(h, sp, None, a_ptr, r_ptr, nr)
            t1 = time.perf_counter()
            rec._chk(code)
            if k >= warm:
                out.append((t1 - t0) * 1000.0)
    finally:
        if gc_was:
            gc.enable()
    return np.array(out)


def run_ours(args):
    import torch
    import paper_2009_00946_b200 as fg

    from paper_2009_00946_b200.replicas import init_replicas
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # init log: communicator size of the per-WFS split
    rc = init_replicas()
    world, rank, local = rc.world, rc.rank, rc.local_rank
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    d = preset_dims(args.preset)
    b = args.precision // 8
    peak, peak_kind = peaks()

    rec = fg.Reconstructor(args.preset, precision=args.precision, batch=1, device=local)
    shard = args.shard and world > 1
    shard_wfs = None
    if shard:
        from paper_2009_00946_b200.replicas import shard_frame
        shard_wfs = shard_frame(rec, rc)
    rec.build_preconditioner()
    F = 16
    # sharded ranks reconstruct the same frame: a common slope stream
    stream_host = slope_stream(rec, args.preset, F, seed=1 if shard else rc.seed)
    stream = torch.from_numpy(stream_host).to(dev)
    st = torch.cuda.Stream(dev)  # a real stream: events, flushes and the graph all order on it
    torch.cuda.set_stream(st)
    rec.set_stream(st.cuda_stream)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    S = d["S"]

    def load(k, r=rec):
        # slopes for frame k into the library's resident slot (outside timing)
        r.load_slopes_device(stream[k % F].data_ptr())

    for k in range(max(args.warmup, 3)):
        load(k)
        rec.step_device(None)
    rec.sync()

    def timed_frames(r, K):
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
        for k in range(K):
            load(k, r)
            flush.zero_()
            starts[k].record(st)
            r.step_device(None)
            ends[k].record(st)
        torch.cuda.synchronize(dev)
        r.sync()
        return np.array([s_.elapsed_time(e_) for s_, e_ in zip(starts, ends)])

    # ---- device-resident timed region (exactly K frames) ----------------------------
    K = args.steps
    rc.barrier()
    torch.cuda.synchronize(dev)
    with Clocks(local) as clk:
        ms = timed_frames(rec, K)
    rc.barrier()
    total_ms = float(ms.sum())
    p50, p99 = float(np.percentile(ms, 50)), float(np.percentile(ms, 99))
    total_ms, p50, p99 = rc.max_over_ranks([total_ms, p50, p99], device=dev)
    value = K / (total_ms / 1000.0) if shard else rc.aggregate_throughput(K, total_ms)

    # ---- latency distribution: >= 1000 frames whatever --steps is (p99 needs them) ----
    NL = max(1000, K)
    lms = timed_frames(rec, NL)
    l50, l99, lmax = rc.max_over_ranks([float(np.percentile(lms, 50)), float(np.percentile(lms, 99)),
                                        float(lms.max())], device=dev)
    latency = {"frames": NL, "p50_ms": round(l50, 5), "p99_ms": round(l99, 5), "max_ms": round(lmax, 5),
               "recon_per_s_p50": round(1000.0 / l50, 1), "l2": "flushed before every frame",
               "note": "separate sample after the timed region, same method; max over ranks"}

    # ---- per-function kernel times inside the frame graph (event nodes) -------------
    def before(f):
        load(f)
        flush.zero_()

    prof, prof_frame_ms = graph_function_profile(rec, 30, before, d, b)
    roof = roofline_object(prof, peak, peak_kind, f"fp{args.precision}",
                           "event-record nodes between the frame graph's launches (telemetry graph, L2 flushed "
                           f"before each frame, 30 frames).  The event nodes serialise the programmatic-launch "
                           f"overlap ({prof_frame_ms:.4f} ms per telemetry frame vs {l50:.4f} ms p50), so shares "
                           "hold and per-launch times are upper bounds")

    # ---- e2e through the C-ABI with host buffers -------------------------------------
    import ctypes as C
    lib = fg.lib()
    dp = C.POINTER(C.c_double)
    pin_s, host_note = host_slope_ring(stream_host, torch)
    pin_a = torch.zeros(d["A"], dtype=torch.float64).pin_memory()
    pin_rho = torch.zeros(d["iters"], dtype=torch.float64).pin_memory()
    a_ptr, r_ptr = C.cast(pin_a.data_ptr(), dp), C.cast(pin_rho.data_ptr(), dp)
    NE = max(1000, min(K, 5000))
    warm_e = max(args.warmup, 3)
    e2e_ms = e2e_loop(rec, lib, [C.cast(pin_s[f].data_ptr(), dp) for f in range(F)], a_ptr, r_ptr, NE, warm_e,
                      flush, dev, torch)
    # the reference's calling convention: slopes in an ordinary (pageable) vector, a^(1) into one
    page_s = np.ascontiguousarray(stream_host.copy())
    page_a, page_r = np.zeros(d["A"]), np.zeros(d["iters"])
    e2e_pg = e2e_loop(rec, lib, [page_s[f].ctypes.data_as(dp) for f in range(F)], page_a.ctypes.data_as(dp),
                      page_r.ctypes.data_as(dp), NE, warm_e, flush, dev, torch)
    e_mean, e_pg_mean, e50, e99, g50, g99 = rc.max_over_ranks(
        [float(np.mean(e2e_ms)), float(np.mean(e2e_pg)), float(np.percentile(e2e_ms, 50)),
         float(np.percentile(e2e_ms, 99)), float(np.percentile(e2e_pg, 50)), float(np.percentile(e2e_pg, 99))],
        device=dev)
    e2e_val = 1000.0 / e_mean if shard else rc.aggregate_throughput(1, e_mean)
    e2e_pg_val = 1000.0 / e_pg_mean if shard else rc.aggregate_throughput(1, e_pg_mean)

    # ---- the north-star per-WFS split at N > 1 (always reported beside the replicas) ---
    shard_info = None
    if world > 1 and not shard:
        try:
            from paper_2009_00946_b200.replicas import shard_frame
            rs = fg.Reconstructor(args.preset, precision=args.precision, batch=1, device=local)
            wfs = shard_frame(rs, rc)
            rs.build_preconditioner()
            rs.set_stream(st.cuda_stream)
            shared = torch.from_numpy(slope_stream(rs, args.preset, F, seed=1)).to(dev)  # one common frame stream
            for k in range(5):
                rs.load_slopes_device(shared[k % F].data_ptr())
                rs.step_device(None)
            rs.sync()
            rc.barrier()
            KS = max(K, 200)
            s0 = [torch.cuda.Event(enable_timing=True) for _ in range(KS)]
            s1 = [torch.cuda.Event(enable_timing=True) for _ in range(KS)]
            for k in range(KS):
                rs.load_slopes_device(shared[k % F].data_ptr())
                flush.zero_()
                s0[k].record(st)
                rs.step_device(None)
                s1[k].record(st)
            torch.cuda.synchronize(dev)
            rs.sync()
            sms = np.array([x.elapsed_time(y) for x, y in zip(s0, s1)])
            sp50, sp99, smean = rc.max_over_ranks([float(np.percentile(sms, 50)), float(np.percentile(sms, 99)),
                                                   float(sms.mean())], device=dev)
            shard_info = {"world": world, "rank0_wfs": list(wfs), "frames": KS, "p50_ms": round(sp50, 5),
                          "p99_ms": round(sp99, 5), "recon_per_s": round(1000.0 / smean, 1),
                          "single_gpu_p50_ms": round(l50, 5), "p99_vs_single_gpu": round(sp99 / l99, 3),
                          "kept": bool(sp99 < l99), "exchange": "ncclAllReduce of the partial adjoint layer sums, "
                                                              "5 per frame, captured in the frame graph",
                          "note": "one instance's frame split by WFS over all ranks (SURVEY 8e); max over ranks"}
            rs.close()
        except Exception as e:  # noqa: BLE001 -- the replicas number above stands on its own
            shard_info = {"world": world, "error": f"{type(e).__name__}: {e}"[:300]}

    # ---- batch-64 throughput (HBM-bound regime) ----------------
    batch_info = None
    if args.batch64 and not shard:
        B = 64
        fb = frame_bytes(d, b) * B
        KB = 30
        plan_b = {}

        def time_split(parts):
            """64 instances per step as `parts` engines of 64/parts on their own streams."""
            nb = B // parts
            engs = []
            for p_ in range(parts):
                r_ = fg.Reconstructor(args.preset, precision=args.precision, batch=nb, device=local)
                r_.build_preconditioner()
                s_ = torch.cuda.Stream(dev)
                r_.set_stream(s_.cuda_stream)
                slab = stream.repeat((B + F - 1) // F, 1)[p_ * nb:(p_ + 1) * nb].contiguous()
                r_.load_slopes_device(slab.data_ptr())
                engs.append((r_, s_, slab))
            for r_, _, _ in engs:
                for _ in range(3):
                    r_.step_device(None)
            torch.cuda.synchronize(dev)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _, s_, _ in engs:
                s_.wait_event(e0)
            for _ in range(KB):
                for r_, _, _ in engs:
                    r_.step_device(None)
            for _, s_, _ in engs:
                ev = torch.cuda.Event()
                ev.record(s_)
                st.wait_event(ev)
            e1.record(st)
            torch.cuda.synchronize(dev)
            prof_b = None
            plan_b.update(engs[0][0].plan_info())
            if parts == 1:  # per-function HBM roofline where the working set exceeds L2
                engs[0][0].set_stream(st.cuda_stream)
                prof_b, _ = graph_function_profile(engs[0][0], 3, lambda f: None, d, b, batch=B)
            for r_, _, _ in engs:
                r_.sync()
                r_.close()
            return e0.elapsed_time(e1) / KB, prof_b

        one, prof_b = time_split(1)
        splits = {1: one}
        for parts in (2, 4, 8):
            splits[parts], _ = time_split(parts)
        best = min(splits, key=splits.get)
        bms = splits[best]
        two = splits[2]
        roof_b = roofline_object(prof_b, peak, peak_kind, f"fp{args.precision}_b64",
                                 "event-record nodes of the 64-instance frame graph (3 frames, working set > L2)")
        batch_info = {"batch": B, "ms_per_step": round(bms, 4), "recon_per_s": round(B * 1000.0 / bms, 1),
                      "roofline_frac_frame_model": round(fb / (bms / 1000.0) / 1e9 / peak, 4),
                      "engines": best,
                      "ms_per_step_1x64": round(one, 4), "ms_per_step_2x32_two_streams": round(two, 4),
                      "ms_per_step_4x16_four_streams": round(splits[4], 4),
                      "ms_per_step_8x8_eight_streams": round(splits[8], 4),
                      "transforms": {2: "whole-layer kernels (one CTA per layer and instance), forward(k) + "
                                        "inverse(k+1) fused in one cluster of the layer CTAs per instance",
                                     1: "whole-layer kernels (one CTA per layer and instance)"}.get(
                          plan_b.get("whole_layer", 0), "cluster kernels"),
                      "roofline": roof_b,
                      "note": "64 instances per step, inputs resident, no flush between steps "
                              "(working set 64 x ~15 MB > L2); best of one 64-instance engine and 2 / 4 / 8 "
                              "engines of 32 / 16 / 8 instances on as many concurrent streams (small engines' "
                              "latency-bound and bandwidth-bound kernels overlap across streams)"}

    # ---- the other BASELINE configs (rank 0, N=1): single-frame latency -------------
    configs = None
    if rank == 0 and world == 1 and not shard and args.configs:
        configs = {}
        for tag, name in (("1_small_mcao_2dm", "small_mcao_2dm"), ("2_elt_ltao84", "elt_ltao84"),
                          ("4_elt_moao84", "elt_moao84")):
            pth = os.path.join(ROOT, "presets", name + ".json")
            dc = preset_dims(pth)
            rx = fg.Reconstructor(pth, precision=args.precision, device=local)
            rx.build_preconditioner()
            rx.set_stream(st.cuda_stream)
            sx = torch.from_numpy(slope_stream(rx, pth, 8, seed=rc.seed)).to(dev)
            for k in range(max(args.warmup, 3)):
                rx.load_slopes_device(sx[k % 8].data_ptr())
                rx.step_device(None)
            rx.sync()
            KC = 1000
            cs = [torch.cuda.Event(enable_timing=True) for _ in range(KC)]
            ce = [torch.cuda.Event(enable_timing=True) for _ in range(KC)]
            for k in range(KC):
                rx.load_slopes_device(sx[k % 8].data_ptr())
                flush.zero_()
                cs[k].record(st)
                rx.step_device(None)
                ce[k].record(st)
            torch.cuda.synchronize(dev)
            rx.sync()
            cms = np.array([a.elapsed_time(e_) for a, e_ in zip(cs, ce)])
            c50 = float(np.percentile(cms, 50))
            fbx = frame_bytes(dc, b)
            configs[tag] = {"preset": os.path.relpath(pth, ROOT), "n_coeff": dc["n"], "n_slopes": dc["S"],
                            "n_act": dc["A"], "frames": KC, "p50_ms": round(c50, 5),
                            "p99_ms": round(float(np.percentile(cms, 99)), 5),
                            "recon_per_s": round(1000.0 / float(np.mean(cms)), 1),
                            "frame_roofline_frac_at_p50": round(fbx / (c50 / 1000.0) / 1e9 / peak, 5)}
            rx.close()

    # ---- CPU baseline (rank 0, N=1 only) -------------------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        from oracle import RefOracle  # noqa: E402
        if RefOracle.available():
            threads = min(max(d["L"], d["W"]), os.cpu_count() or 1)
            frames = args.cpu_frames
            us, thr = cpu_reference_time(args.preset, stream_host, frames, threads)
            cms = us / 1000.0
            cpu = {"value": round(1000.0 / float(np.mean(cms)), 3), "unit": UNIT, "cores": thr, "kind": "reference",
                   "cpu_model": cpu_model(), "nproc": os.cpu_count(),
                   "sample": f"{frames} frames of the reference Reconstructor::step (oracle/_ref, L=M shadow preset) "
                             f"on this slope stream, {thr} pool threads (min(max(L,W), nproc)), {os.cpu_count()} host "
                             f"cpus ({cpu_model()}); p50 {np.percentile(cms, 50):.2f} ms p99 "
                             f"{np.percentile(cms, 99):.2f} ms"}

    if rank == 0:
        fb = frame_bytes(d, b)
        launches = rec.launches_per_step()
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world, "steps": K,
            "warmup": args.warmup, "ms_per_step": round(total_ms / K, 5), "p50_ms": round(p50, 5),
            "p99_ms": round(p99, 5), "higher_is_better": True, "scaling": "strong" if shard else "weak",
            "vs_baseline": None,
            "dtype": "f64" if args.precision == 64 else "f32", "data": "synthetic",
            "config": {"workload": "ELT MCAO-84 (BASELINE config 3: 84x84 SH, 6 LGS + 3 NGS, 9 layers, 3 DMs), "
                                   "1 instance/rank, closed loop, 4 PCG iters, single-frame latency",
                       "preset": os.path.relpath(args.preset, ROOT), "n_coeff": d["n"], "n_slopes": S,
                       "n_act": d["A"], "l2": "flushed (256 MiB write) before every timed frame",
                       "parallelism": (f"wfs-shard x{world} (rank 0 owns WFS {shard_wfs})" if shard
                                       else f"replicas x{world}")},
            "latency": latency,
            "frame_roofline": {"bytes_per_frame": fb, "achieved_gbs": round(fb / (l50 / 1000.0) / 1e9, 2),
                               "frac_at_p50": round(fb / (l50 / 1000.0) / 1e9 / peak, 5),
                               "roofline_us": round(fb / (peak * 1e9) * 1e6, 3)},
            "roofline": roof,
            "e2e": {"value": round(e2e_val, 3), "unit": UNIT, "h2d_bytes_per_step": S * 8, "host_buffers": host_note,
                    "d2h_bytes_per_step": d["A"] * 8 + d["iters"] * 8 + 8, "frames": NE,
                    "p50_ms": round(e50, 5), "p99_ms": round(e99, 5),
                    "pageable": {"value": round(e2e_pg_val, 3), "unit": UNIT, "p50_ms": round(g50, 5),
                                 "p99_ms": round(g99, 5),
                                 "host_buffers": "ordinary numpy arrays (pageable), as the reference's "
                                                 "span<const double> over a std::vector"}},
            "gpu_launches": launches * K,
            "clocks": clk.summary(),
        }
        if shard_info:
            line["shard"] = shard_info
        if cpu:
            line["cpu_baseline"] = cpu
        if batch_info:
            line["batch64"] = batch_info
        if configs:
            line["other_configs"] = configs
        print(json.dumps(line))
    rc.shutdown()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--precision", type=int, default=64, choices=[64, 32])
    ap.add_argument("--preset", default=DEFAULT_PRESET)
    ap.add_argument("--cpu-frames", type=int, default=150)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-batch64", dest="batch64", action="store_false")
    ap.add_argument("--no-configs", dest="configs", action="store_false",
                    help="skip the single-frame latency of BASELINE configs 1, 2 and 4")
    ap.add_argument("--shard", action="store_true", help="N>1: per-WFS sharding of one frame (NCCL exchange)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
