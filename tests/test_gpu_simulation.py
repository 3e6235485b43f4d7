"""GPU parity of the closed-loop simulation harness: measurement
synthesis through the device forward model and the whole run_closed_loop
(simulation.hpp:321-345) on the device reconstructor, against the unmodified
reference run in-process (oracle/_ref).  Tolerances: the north star's 1e-9
(fp64) on the loop's outputs; the slopes themselves within 1e-12."""
import json

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


@pytest.mark.parametrize("name", ["small_mcao", "elt_mcao84"])
def test_synthesis_matches_reference(name, tmp_path):
    path = _windy(tmp_path, name) if name == "small_mcao" else preset(name + ".json")
    o = RefOracle(path)
    geo = sim.SimGeometry.load(path)
    rec = fg.Reconstructor(path)
    truth = sim.generate_atmosphere(geo, 9)
    A = sum(n * n for n, _h, _e in geo.dms)
    a = 0.2 * np.random.default_rng(1).standard_normal(A)
    for k in (0, 3):
        got = sim.synthesize(rec, geo, sim.truth_at_step(geo, truth, k), a, sim.splitmix64(9 + k))
        assert rel_err(got, o.synthesize(9, k, a)) <= 1e-12, k


@pytest.mark.parametrize("name,steps", [("small_mcao", 6), ("small_mcao_windy", 6), ("elt_mcao84", 2)])
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
