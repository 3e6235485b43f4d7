"""CPU parity of the simulation harness's host parts (paper_2009_00946_b200/
simulation.py) against the unmodified reference (oracle/_ref): the random
streams, the truth screens, frozen flow and the quality metrics.  The device
parts (slopes, loop) are in tests/test_gpu_simulation.py."""
import json

import numpy as np
import pytest

from conftest import preset
from oracle import RefOracle, rel_err
from paper_2009_00946_b200 import simulation as sim

pytestmark = pytest.mark.skipif(not RefOracle.available(), reason="oracle/_ref not built")


def test_mt19937_64_matches_the_standard():
    # [rand.predef]: the 10000th invocation of a default-constructed mt19937_64
    assert int(sim.MT19937_64(5489).draws(10000)[-1]) == 9981545732273789042


@pytest.mark.parametrize("seed", [0, 7, sim.splitmix64(12345)])
def test_gaussian_stream_matches_reference(seed):
    ref = RefOracle.gauss(seed, 2001)
    g = sim.GaussianStream(seed)
    got = np.concatenate([g.take(1), g.take(1000), g.take(1000)])  # odd split exercises the cached pair half
    np.testing.assert_allclose(got, ref, rtol=1e-14, atol=1e-15)


@pytest.mark.parametrize("name", ["mini", "small_mcao", "elt_mcao84"])
def test_atmosphere_matches_reference(name):
    o = RefOracle(preset(name + ".json"))
    geo = sim.SimGeometry.load(preset(name + ".json"))
    for seed in (1, 17):
        got = np.concatenate([l.ravel() for l in sim.generate_atmosphere(geo, seed)])
        assert rel_err(got, o.atmosphere(seed)) <= 1e-12


def _windy(tmp_path, base="small_mcao"):
    j = json.load(open(preset(base + ".json")))
    j["simulation"]["wind_m_per_step"] = [[0.35, -0.2], [-0.7, 0.45], [1.3, 0.9]][:len(j["layers"])]
    p = tmp_path / "windy.json"
    p.write_text(json.dumps(j))
    return str(p)


def test_frozen_flow_matches_reference(tmp_path):
    path = _windy(tmp_path)
    o = RefOracle(path)
    geo = sim.SimGeometry.load(path)
    truth = sim.generate_atmosphere(geo, 3)
    for k in (0, 1, 5, 40):
        got = np.concatenate([l.ravel() for l in sim.truth_at_step(geo, truth, k)])
        assert rel_err(got, o.truth_at_step(3, k)) <= 1e-12, k


@pytest.mark.parametrize("name", ["small_mcao", "elt_mcao84"])
def test_quality_matches_reference(name):
    o = RefOracle(preset(name + ".json"))
    geo = sim.SimGeometry.load(preset(name + ".json"))
    truth = sim.generate_atmosphere(geo, 5)
    rng = np.random.default_rng(0)
    A = sum(n * n for n, _h, _e in geo.dms)
    for dm in (np.zeros(A), 0.3 * rng.standard_normal(A)):
        q = sim.evaluate_quality(geo, truth, dm)
        fr, le, rms = o.quality(np.concatenate([l.ravel() for l in truth]), dm)
        assert abs(q.field_rms - fr) <= 1e-12 * fr
        assert abs(q.layer_rel_err - le) <= 1e-12 * max(le, 1e-300)
        np.testing.assert_allclose(q.rms_per_dir, rms[:q.rms_per_dir.size], rtol=1e-12)
