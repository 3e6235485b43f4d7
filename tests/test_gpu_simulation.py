"""GPU parity of the device closed-loop simulation harness against
the unmodified reference run in-process (oracle/_ref): the random streams, the
truth screens and frozen flow, measurement synthesis, the quality metrics and
the whole run_closed_loop (simulation.hpp:40-345).  Tolerances: the north star's
1e-9 (fp64) on the loop's outputs; every building block within 1e-12."""
import json
import time

import numpy as np
import pytest

import paper_2009_00946_b200 as fg
from conftest import preset
from oracle import RefOracle, rel_err
from paper_2009_00946_b200 import simulation as sim

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not RefOracle.available(), reason="oracle/_ref not built")]


def _windy(tmp_path, base):
    j = json.load(open(preset(base + ".json")))
    j["simulation"]["wind_m_per_step"] = [[0.35, -0.2], [-0.7, 0.45], [1.3, 0.9]][:len(j["layers"])]
    p = tmp_path / f"{base}_windy.json"
    p.write_text(json.dumps(j))
    return str(p)


@pytest.mark.parametrize("seed", [0, 7, sim.splitmix64(12345)])
def test_gaussian_stream_matches_reference(seed):
    """k_gauss (one warp per mt19937_64 stream + Box-Muller) against GaussianStream."""
    ref = RefOracle.gauss(seed, 2000)
    np.testing.assert_allclose(sim.gaussian_stream(seed, 2000), ref, rtol=1e-14, atol=1e-15)


@pytest.mark.parametrize("name", ["mini", "small_mcao", "elt_mcao84"])
def test_atmosphere_matches_reference(name):
    o = RefOracle(preset(name + ".json"))
    rec = fg.Reconstructor(preset(name + ".json"))
    for seed in (1, 17):
        assert rel_err(sim.generate_atmosphere(rec, seed), o.atmosphere(seed)) <= 1e-12, seed


def test_frozen_flow_matches_reference(tmp_path):
    path = _windy(tmp_path, "small_mcao")
    o = RefOracle(path)
    rec = fg.Reconstructor(path)
    for k in (0, 1, 5, 40):
        assert rel_err(sim.generate_atmosphere(rec, 3, k), o.truth_at_step(3, k)) <= 1e-12, k


@pytest.mark.parametrize("name", ["small_mcao", "elt_mcao84"])
def test_synthesis_matches_reference(name, tmp_path):
    path = _windy(tmp_path, name) if name == "small_mcao" else preset(name + ".json")
    o = RefOracle(path)
    rec = fg.Reconstructor(path)
    a = 0.2 * np.random.default_rng(1).standard_normal(rec.dims.A)
    for k in (0, 3):
        got = sim.synthesize(rec, sim.generate_atmosphere(rec, 9, k), a, sim.splitmix64(9 + k))
        assert rel_err(got, o.synthesize(9, k, a)) <= 1e-12, k


@pytest.mark.parametrize("name", ["small_mcao", "elt_mcao84"])
def test_quality_matches_reference(name):
    o = RefOracle(preset(name + ".json"))
    rec = fg.Reconstructor(preset(name + ".json"))
    truth = sim.generate_atmosphere(rec, 5)
    rng = np.random.default_rng(0)
    for dm in (np.zeros(rec.dims.A), 0.3 * rng.standard_normal(rec.dims.A)):
        q = sim.evaluate_quality(rec, truth, dm)
        fr, le, rms = o.quality(truth, dm)
        assert abs(q.field_rms - fr) <= 1e-12 * fr
        assert abs(q.layer_rel_err - le) <= 1e-12 * max(le, 1e-300)
        np.testing.assert_allclose(q.rms_per_dir, rms[:q.rms_per_dir.size], rtol=1e-12)


@pytest.mark.parametrize("name,steps", [("small_mcao", 6), ("small_mcao_windy", 6), ("elt_mcao84", 4)])
def test_closed_loop_matches_reference(name, steps, tmp_path):
    path = _windy(tmp_path, "small_mcao") if name == "small_mcao_windy" else preset(name + ".json")
    ref = RefOracle(path).run_closed_loop(steps, atm=1, noise=2, threads=0)
    got = sim.run_closed_loop(path, steps, atmosphere_seed=1, noise_seed=2)
    fr = np.array([q.field_rms for q in got.records])
    le = np.array([q.layer_rel_err for q in got.records])
    rho = np.stack([q.rho for q in got.records])
    assert rel_err(fr, ref["field_rms"]) <= 1e-9
    assert rel_err(le, ref["layer_rel_err"]) <= 1e-9
    assert rel_err(rho, ref["rho"]) <= 1e-9
    assert abs(got.uncorrected_field_rms - ref["uncorrected_field_rms"]) <= 1e-9 * ref["uncorrected_field_rms"]
    assert abs(got.final_field_rms - ref["final_field_rms"]) <= 1e-9 * ref["final_field_rms"]
    if name == "small_mcao":
        # the static loop corrects (test_simulation.cpp:245-261 spirit; 6 steps of a 2-step-delay, gain-0.4 loop)
        assert got.final_field_rms < 0.9 * got.uncorrected_field_rms


def test_lnem_loop_runs_on_device():
    """The L != M presets (not runnable by the reference) close the loop too."""
    r = sim.run_closed_loop(preset("small_mcao_2dm.json"), 6)
    assert r.final_field_rms < 0.95 * r.uncorrected_field_rms
    assert all(np.isnan(q.layer_rel_err) for q in r.records)


def test_long_elt_loop_on_device(tmp_path):
    """A long windy ELT closed loop (200 frames) entirely on the device: every
    record finite, its first frames equal the reference's own run of the same
    loop (the records of step k do not depend on the run length), the handle keeps
    stepping afterwards, and the run costs well under a millisecond of wall time
    per frame (no per-frame host round trip)."""
    j = json.load(open(preset("elt_mcao84.json")))
    j["simulation"]["wind_m_per_step"] = [[0.3 * (1 + l % 3), -0.2 * (l % 2)] for l in range(len(j["layers"]))]
    p = tmp_path / "elt_windy.json"
    p.write_text(json.dumps(j))
    rec = fg.Reconstructor(str(p))
    sim.run_closed_loop(str(p), 3, rec=rec)  # warm: tables, graph, preconditioner
    t0 = time.perf_counter()
    r = sim.run_closed_loop(str(p), 200, rec=rec)
    wall = time.perf_counter() - t0
    fr = np.array([q.field_rms for q in r.records])
    assert np.all(np.isfinite(fr))
    ref = RefOracle(str(p)).run_closed_loop(3, atm=1, noise=2, threads=0)
    assert rel_err(fr[:3], ref["field_rms"]) <= 1e-9
    assert wall / 200 < 1e-3, wall
    rec.step(np.zeros(rec.dims.S))
