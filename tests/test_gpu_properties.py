"""The reference's solver-property tests, restated on the GPU path.

Each test cites the reference test it restates (proj/tests/test_reconstructor.cpp,
proj/tests/acceptance_main.cpp).  Where the reference drives pcg_solve directly
on an arbitrary right-hand side, the same solve runs here through the frame:
an open-loop engine whose state is seeded with c = 0, b = 0, r = b_target, p = q
= 0 and fresh scalars, fed zero slopes, performs exactly the reference's
pcg_solve(M, J, c, r, p, q, scalars, iters) on b_target (the RHS update r +=
b1 - b adds 0; reconstructor.hpp:316-323).  The MAORY presets are replayed
against the unmodified reference itself (oracle/_ref) where it is built.
"""
import json

import numpy as np
import pytest

import paper_2009_00946_b200 as fg
from conftest import preset
from oracle import Oracle, RefOracle, rel_err
from test_gpu_parity import smooth_layers

pytestmark = pytest.mark.gpu


def _mini(tmp_path, name="mini", **solver):
    j = json.load(open(preset("mini.json")))
    loop = solver.pop("loop", None)
    gain = solver.pop("gain", None)
    dms = solver.pop("n_act", None)
    j["solver"].update(solver)
    if loop is not None:
        j["loop"]["mode"] = loop
    if gain is not None:
        j["loop"]["gain"] = gain
    if dms is not None:
        for d in j["dms"]:
            d["n_act"] = dms
    p = tmp_path / f"{name}.json"
    p.write_text(json.dumps(j))
    return str(p)


def _dense_M(g):
    n = g.dims.n
    return np.asarray(g.apply_M(np.eye(n))).reshape(n, n).T  # column k = M e_k


def _seed_solve(g, b):
    """State for pcg_solve(M, J, c=0, r=b, p=0, q=0, fresh) through the frame."""
    st = g.get_state()
    for k in ("c", "b", "p", "q"):
        st[k] = np.zeros(g.dims.n)
    st["r"] = np.asarray(b, np.float64).copy()
    st["scalars"] = np.array([0.0, 0.0, 1.0])
    g.set_state(st)


# ---- apply_M / build_rhs ----------------------------------------------------------

@pytest.mark.parametrize("name", ["mini", "maory", "maory9", "elt_mcao84"])
def test_M_symmetric_positive_definite(name):
    """ApplyM.SymmetricPositiveDefiniteRandomized (test_reconstructor.cpp:204-218) and
    acceptance criterion 3 on every shipped config (acceptance_main.cpp:95-120):
    |<Mx,y> - <x,My>| <= 1e-10 |Mx||y| and <Mx,x> > 0 over 20 trials; M 0 = 0."""
    g = fg.Reconstructor(preset(name + ".json"))
    n = g.dims.n
    rng = np.random.default_rng(77)
    x, y = rng.standard_normal((20, n)), rng.standard_normal((20, n))
    mx, my = g.apply_M(x), g.apply_M(y)
    for t in range(20):
        sym = abs(mx[t] @ y[t] - x[t] @ my[t]) / (np.linalg.norm(mx[t]) * np.linalg.norm(y[t]))
        assert sym <= 1e-10, (t, sym)
        assert mx[t] @ x[t] > 0.0
    assert not np.any(g.apply_M(np.zeros(n)))  # ApplyM.ZeroInputGivesZeroOutput (:197-202)


def test_build_rhs_zero_and_linearity():
    """BuildRhs.ZeroAndLinearity (test_reconstructor.cpp:233-249)."""
    g = fg.Reconstructor(preset("mini.json"))
    assert not np.any(g.build_rhs(np.zeros(g.dims.S)))
    s1 = np.random.default_rng(5).standard_normal(g.dims.S)
    b1, b2 = g.build_rhs(s1), g.build_rhs(2.0 * s1)
    assert np.all(np.abs(b2 - 2.0 * b1) <= 1e-14 * np.abs(b1) + 1e-300)


# ---- pcg_solve ---------------------------------------------------------------------

def test_pcg_matches_dense_cholesky(tmp_path):
    """Pcg.MiniSystemMatchesDenseCholesky (test_reconstructor.cpp:121-136) and
    acceptance criterion 4: 50 cold iterations, |r|/|b| < 1e-6 and c within 1e-6
    of the dense Cholesky solve of the matrix assembled from apply_M."""
    g = fg.Reconstructor(_mini(tmp_path, pcg_max_iter=50, loop="open"))
    n = g.dims.n
    M = _dense_M(g)
    b = np.random.default_rng(3).standard_normal(n)
    _seed_solve(g, b)
    g.step(np.zeros(g.dims.S))
    st = g.get_state()
    assert np.linalg.norm(st["r"]) / np.linalg.norm(b) < 1e-6
    L = np.linalg.cholesky(M)
    direct = np.linalg.solve(L.T, np.linalg.solve(L, b))
    assert rel_err(st["c"], direct) < 1e-6


def test_pcg_error_energy_norm_decreases_every_iteration(tmp_path):
    """Pcg.ErrorEnergyNormDecreasesEveryIteration (test_reconstructor.cpp:138-165):
    one iteration per frame with carried scalars (pcg_max_iter = 1) reproduces the
    50-iteration trajectory; the M-norm of the error never grows."""
    g = fg.Reconstructor(_mini(tmp_path, pcg_max_iter=1, loop="open"))
    n = g.dims.n
    M = _dense_M(g)
    b = np.random.default_rng(3).standard_normal(n)
    exact = np.linalg.solve(M, b)
    _seed_solve(g, b)
    prev = 0.0
    for it in range(50):
        g.step(np.zeros(g.dims.S))
        err = g.get_state()["c"] - exact
        energy = np.sqrt(max(0.0, err @ (M @ err)))
        if it > 0 and prev > 1e-12 * np.linalg.norm(exact):
            assert energy <= prev * (1.0 + 1e-13), it
        prev = energy
    # the same 50 iterations in one solve land on the same point
    g50 = fg.Reconstructor(_mini(tmp_path, "m50", pcg_max_iter=50, loop="open"))
    _seed_solve(g50, b)
    g50.step(np.zeros(g.dims.S))
    assert rel_err(g50.get_state()["c"], g.get_state()["c"]) < 1e-10


def test_solution_error_decreases_with_iteration_count(tmp_path):
    """Pcg.SolutionErrorDecreasesWithIterationCount (test_reconstructor.cpp:171-195):
    error against the dense solve is monotone over 4 -> 8 -> 16 iterations, on the
    RHS of a synthetic atmosphere's noiseless slopes."""
    g0 = fg.Reconstructor(preset("mini.json"))
    o = Oracle(preset("mini.json"))
    meas = g0.forward_slopes(smooth_layers(o, 4))
    b = g0.build_rhs(meas)
    exact = np.linalg.solve(_dense_M(g0), b)
    prev = np.inf
    for iters in (4, 8, 16):
        g = fg.Reconstructor(_mini(tmp_path, f"m{iters}", pcg_max_iter=iters, loop="open"))
        _seed_solve(g, b)
        g.step(np.zeros(g.dims.S))
        err = rel_err(g.get_state()["c"], exact)
        assert err < prev, iters
        prev = err


# ---- Reconstructor::step -------------------------------------------------------------

@pytest.mark.parametrize("loop", ["closed", "open"])
def test_zero_gain_holds_the_mirror(loop, tmp_path):
    """ReconstructStep.ZeroGainHoldsTheMirror (test_reconstructor.cpp:255-269)."""
    g = fg.Reconstructor(_mini(tmp_path, loop=loop, gain=0.0))
    st = g.get_state()
    st["a_prev"] = np.full(g.dims.A, 0.25)
    g.set_state(st)
    a1 = g.step(np.random.default_rng(9).standard_normal(g.dims.S))
    assert np.all(a1 == 0.25)


def test_open_loop_unit_gain_returns_fitted_shapes(tmp_path):
    """ReconstructStep.OpenLoopUnitGainReturnsFittedShapes (test_reconstructor.cpp:271-285):
    a^(1) = fit_to_mirrors(st.c) (EXPECT_DOUBLE_EQ: within 4 ulp)."""
    g = fg.Reconstructor(_mini(tmp_path, loop="open", gain=1.0))
    a1 = g.step(np.random.default_rng(13).standard_normal(g.dims.S))
    fit = g.fit(g.coeffs())
    assert np.all(np.abs(a1 - fit) <= 4 * np.spacing(np.maximum(np.abs(a1), np.abs(fit))))


def test_static_atmosphere_warm_restart_converges(tmp_path):
    """ReconstructStep.StaticAtmosphereWarmRestartConverges (test_reconstructor.cpp:
    362-386): fixed noiseless slopes, open loop, 10 warm-restarted frames of 4
    iterations: rho_0 never grows and |r| < 1e-8 |b| at the end."""
    g = fg.Reconstructor(_mini(tmp_path, loop="open"))
    o = Oracle(preset("mini.json"))
    meas = g.forward_slopes(smooth_layers(o, 1))
    prev, b_norm = 0.0, 0.0
    for step in range(10):
        g.step(meas)
        rho0 = g.last_rho[0]
        if step == 0:
            b_norm = np.linalg.norm(g.get_state()["b"])
        else:
            assert rho0 <= prev * (1.0 + 1e-13), step
        prev = rho0
    assert np.linalg.norm(g.get_state()["r"]) < 1e-8 * b_norm


def test_fit_identity_and_coarser_actuator_grid(tmp_path):
    """FitToMirrors.IdentityWhenGridsCoincide / ResamplesOntoCoarserActuatorGrid
    (test_reconstructor.cpp:404-439): n_act = 2^J copies W^-1 c; n_act = 5 samples
    it bilinearly at -e/2 + j e/4 (bilinear_sample, operators.hpp:123-127)."""
    g = fg.Reconstructor(preset("mini.json"))
    c = np.random.default_rng(31).standard_normal(g.dims.n)
    a = g.fit(c)
    phi = g.wavelet(c, True)
    assert np.array_equal(a, phi)  # 8x8 layers, 8x8 DMs
    g5 = fg.Reconstructor(_mini(tmp_path, "m5", n_act=5))
    _, dext, _ = g5.geometry()
    a5 = g5.fit(c).reshape(len(dext), 5, 5)
    for l in range(len(dext)):
        grid = phi[l * 64:(l + 1) * 64].reshape(8, 8)
        e = dext[l]
        for i in range(5):
            for j in range(5):
                u = (-e / 2 + j * e / 4 + e / 2) / (e / 7)
                v = (-e / 2 + i * e / 4 + e / 2) / (e / 7)
                j0, i0 = min(int(np.floor(u)), 6), min(int(np.floor(v)), 6)
                fx, fy = u - j0, v - i0
                want = ((1 - fy) * (1 - fx) * grid[i0, j0] + (1 - fy) * fx * grid[i0, j0 + 1] +
                        fy * (1 - fx) * grid[i0 + 1, j0] + fy * fx * grid[i0 + 1, j0 + 1])
                assert abs(a5[l, i, j] - want) <= 1e-14 * max(1.0, abs(want)), (l, i, j)


# ---- the shipped MAORY presets against the live reference ------------------------------

@pytest.mark.skipif(not RefOracle.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("name", ["maory", "maory9"])
def test_maory_presets_replay_live_reference(name):
    """Acceptance criterion 8's workload (acceptance_main.cpp:207-226): the
    reference's own closed loop on a shipped MAORY preset (run_bench's stream,
    bench.hpp:144-154: its atmosphere, its noise, its a^(-1) feedback), recorded
    from the unmodified reference and replayed on the GPU: c, a^(1) and rho per
    frame within 1e-9; and the reference's preconditioner within 1e-12."""
    path = preset(name + ".json")
    ref = RefOracle(path)
    ref.build_preconditioner()
    meas, c, a, rho, _ = ref.record(seed=3, frames=5)
    g = fg.Reconstructor(path)
    assert rel_err(g.preconditioner(), ref.preconditioner()) <= 1e-12
    for k in range(meas.shape[0]):
        ak = g.step(meas[k])
        assert rel_err(g.coeffs(), c[k]) <= 1e-9, ("c", k)
        assert rel_err(ak, a[k]) <= 1e-9, ("a", k)
        assert rel_err(g.last_rho, rho[k]) <= 1e-9, ("rho", k)


# ---- acceptance criteria 1, 2, 6, 9 (acceptance_main.cpp:62-268) ------------------------

def _adjoint_defect(ax, y, x, aty):
    """verify.hpp:75-83: |<Ax,y> - <x,A^T y>| over 0.5 (|Ax||y| + |x||A^T y|)."""
    lhs, rhs = ax @ y, x @ aty
    scale = 0.5 * (np.linalg.norm(ax) * np.linalg.norm(y) + np.linalg.norm(x) * np.linalg.norm(aty))
    return abs(lhs - rhs) / scale if scale else abs(lhs - rhs)


@pytest.mark.parametrize("name", ["mini", "small_mcao", "elt_mcao84"])
def test_adjoint_identities_randomized(name):
    """Criterion 2 (acceptance_main.cpp:62-95, verify.hpp:192-211): Gamma/Gamma^T,
    P/P^T (the hot path's separable gather) and W^-1/W^-T (= W: orthonormal) are
    adjoint pairs at 1e-12 over randomized trials (1000 on mini as the reference,
    200 at the larger scales), every trial batched through one call per operator."""
    g = fg.Reconstructor(preset(name + ".json"))
    d = g.dims
    trials = 1000 if name == "mini" else 200
    rng = np.random.default_rng(2)
    worst = {}
    for op, fwd, adj, nin, nout in (("sh", g.sh, g.sh_transpose, d.Nw, d.S),
                                    ("propagation", g.propagate, g.propagate_transpose, d.n, d.Nw),
                                    ("wavelet", lambda v: g.wavelet(v, True), lambda v: g.wavelet(v, False), d.n, d.n)):
        x, y = rng.standard_normal((trials, nin)), rng.standard_normal((trials, nout))
        ax, aty = np.atleast_2d(fwd(x)), np.atleast_2d(adj(y))
        worst[op] = max(_adjoint_defect(ax[t], y[t], x[t], aty[t]) for t in range(trials))
    assert all(v <= 1e-12 for v in worst.values()), worst


def test_dense_operators_match_the_reference_matrices():
    """Criterion 1 (acceptance_main.cpp:62-83): the matrix-free M assembled densely
    on the mini config equals the reference's (the oracle's, pinned bitwise to the
    reference) at 1e-10, and so does the RHS map assembled from unit slopes."""
    g = fg.Reconstructor(preset("mini.json"))
    o = Oracle(preset("mini.json"))
    d = g.dims
    eye = np.eye(d.n)
    Mg = np.atleast_2d(g.apply_M(eye))
    Mo = np.stack([o.apply_M(eye[k]) for k in range(d.n)])
    assert rel_err(Mg, Mo) <= 1e-10
    es = np.eye(d.S)[:64]
    Bg = np.atleast_2d(g.build_rhs(es))
    Bo = np.stack([o.build_rhs(es[k]) for k in range(es.shape[0])])
    assert rel_err(Bg, Bo) <= 1e-10


def test_noiseless_closed_loop_corrects_below_ten_percent(tmp_path):
    """Criterion 6 (acceptance_main.cpp:155-168): the noiseless mini loop at gain 0.4,
    4 PCG iterations, 20 steps ends below 10 % of the uncorrected field RMS --
    run entirely on the device (fewha_gpu_run_closed_loop)."""
    from paper_2009_00946_b200 import simulation as sim

    j = json.load(open(preset("mini.json")))
    j["simulation"]["noise"] = False
    j["loop"]["gain"] = 0.4
    j["solver"]["pcg_max_iter"] = 4
    p = tmp_path / "mini_noiseless.json"
    p.write_text(json.dumps(j))
    r = sim.run_closed_loop(str(p), 20)
    assert r.final_field_rms / r.uncorrected_field_rms < 0.10, (r.final_field_rms, r.uncorrected_field_rms)


@pytest.mark.parametrize("order", range(1, 11))
def test_wavelet_properties_across_scales_and_orders(order, tmp_path):
    """Criterion 9 (acceptance_main.cpp:228-268): for J = 3..7 (one layer each) and
    this Daubechies order: the cluster transforms are orthonormal (1e-12), W^-1 W x
    reconstructs x (1e-10 of max|x|), and a constant c maps to 2^J c at the coarse
    coefficient with every detail below 1e-12 c 2^J."""
    j = json.load(open(preset("mini.json")))
    base = j["layers"][0]
    j["layers"] = [dict(base, grid_order=J, height=1000.0 * i, relative_strength=0.2) for i, J in enumerate(range(3, 8))]
    j["dms"] = [{"n_act": 1 << J, "conjugation_height": 1000.0 * i} for i, J in enumerate(range(3, 8))]
    j["solver"]["wavelet_order"] = order
    p = tmp_path / f"wav{order}.json"
    p.write_text(json.dumps(j))
    g = fg.Reconstructor(str(p))
    rng = np.random.default_rng(order)
    x = rng.standard_normal(g.dims.n)
    offs = np.cumsum([0] + [(1 << J) ** 2 for J in range(3, 8)])
    wx = g.wavelet(x, False)
    rec = g.wavelet(wx, True)
    for l, J in enumerate(range(3, 8)):
        a, b = offs[l], offs[l + 1]
        assert abs(np.linalg.norm(wx[a:b]) / np.linalg.norm(x[a:b]) - 1.0) <= 1e-12, J
        assert np.max(np.abs(rec[a:b] - x[a:b])) <= 1e-10 * np.max(np.abs(x[a:b])), J
    c = 0.8125
    wc = g.wavelet(np.full(g.dims.n, c), False)
    for l, J in enumerate(range(3, 8)):
        blk = wc[offs[l]:offs[l + 1]]
        n = 1 << J
        assert abs(blk[0] - c * n) <= 1e-12 * c * n, J
        assert np.max(np.abs(blk[1:])) <= 1e-12 * c * n, J
