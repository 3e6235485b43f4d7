"""GPU tests of the per-WFS sharded frame.

Shard r of `world` owns a contiguous WFS range; the partial adjoint layer sums
are exchanged after the RHS and after every apply_M.  On one GPU the exchange
is exercised two ways:
  * in-process groups (fewha_gpu_group_step_device): members on one device, the
    exchange a fixed rank-order sum kernel over the members' partial buffers --
    the same kernel reads peers over NVLink when members sit on different GPUs;
  * the NCCL path at world 1 (the frame graph captures ncclAllReduce).
Tolerances are the north star's (fp64 1e-9, fp32 1e-4) against the oracle; the
replicated state must be bitwise identical on every member.
"""
import numpy as np
import pytest

import paper_2009_00946_b200 as fg
from conftest import preset
from oracle import Oracle, rel_err
from test_gpu_parity import STEP_TOL, noisy_slopes, smooth_layers

pytestmark = pytest.mark.gpu


def _group(path, world, precision):
    members = [fg.Reconstructor(path, precision=precision) for _ in range(world)]
    for r, m in enumerate(members):
        m.shard(r, world)
        assert m.shard_wfs() == fg.shard_range(path, r, world)
        m.build_preconditioner()
    return members


@pytest.mark.parametrize("name,world,precision", [
    ("small_mcao", 2, 64), ("small_mcao", 3, 64), ("elt_mcao84_3dm", 2, 64), ("elt_mcao84_3dm", 4, 64),
    ("elt_mcao84_3dm", 2, 32), ("elt_moao84", 3, 64)])
def test_group_frames_match_oracle(name, world, precision):
    path = preset(name + ".json")
    o = Oracle(path)
    o.build_preconditioner()
    members = _group(path, world, precision)
    lay = smooth_layers(o, 7)
    tol = STEP_TOL[precision]
    for k in range(3):
        st = o.get_state()
        s = noisy_slopes(o, lay, 300 + k, st["a_prev2"] if o.g["loop_closed"] else None)
        for m in members:
            m.load_slopes(s)
        fg.group_step_device(members)
        for m in members:
            m.sync()
        c_o, a_o, _ = o.step(s)
        states = [m.get_state() for m in members]
        for key in ("c", "r", "p", "q", "a_prev"):  # replicated state: bitwise equal on every member
            for st_m in states[1:]:
                assert np.array_equal(st_m[key], states[0][key]), (key, k)
        assert rel_err(states[0]["c"], c_o) <= tol, ("c", k, rel_err(states[0]["c"], c_o))
        assert rel_err(states[0]["a_prev"], a_o) <= tol, ("a", k, rel_err(states[0]["a_prev"], a_o))


def test_group_matches_unsharded_engine():
    """Sharding changes only the summation order of the adjoint layer sums."""
    path = preset("elt_mcao84_3dm.json")
    ref = fg.Reconstructor(path)
    ref.build_preconditioner()
    members = _group(path, 3, 64)
    o = Oracle(path)
    lay = smooth_layers(o, 9)
    for k in range(3):
        s = noisy_slopes(o, lay, 400 + k, ref.get_state()["a_prev2"])
        a_ref = ref.step(s)
        for m in members:
            m.load_slopes(s)
        fg.group_step_device(members)
        members[0].sync()
        st = members[0].get_state()
        assert rel_err(st["a_prev"], a_ref) <= 1e-10
        assert rel_err(st["c"], ref.coeffs()) <= 1e-10


def test_nccl_world1_is_bitwise_the_unsharded_frame():
    """The NCCL exchange path (graph-captured ncclAllReduce) at world 1."""
    path = preset("elt_mcao84_3dm.json")
    ref = fg.Reconstructor(path)
    ref.build_preconditioner()
    sh = fg.Reconstructor(path)
    sh.shard(0, 1, fg.nccl_unique_id())
    sh.build_preconditioner()
    rng = np.random.default_rng(3)
    for k in range(3):
        s = rng.standard_normal(ref.dims.S) * 0.01
        a0 = ref.step(s)
        a1 = sh.step(s)
        assert np.array_equal(a0, a1), k
        assert np.array_equal(ref.coeffs(), sh.coeffs()), k


def test_group_member_refuses_standalone_step():
    path = preset("small_mcao.json")
    m = _group(path, 2, 64)[0]
    with pytest.raises(fg.ArgumentError, match="group"):
        m.step(np.zeros(m.dims.S))


@pytest.mark.parametrize("devices", [[0], [0, 0], [0, 0, 0]])
def test_multi_device_handle_steps_like_one_reconstructor(devices):
    """fewha_gpu_create_multi (SURVEY 8(b)'s devices/n_devices form): one handle over
    the listed devices -- a per-WFS shard group when there are several -- driven
    through the ordinary fewha_gpu_step: a^(1), st.c and rho match the oracle at
    1e-9 over closed-loop frames, and reset / set_state act on every shard."""
    path = preset("elt_mcao84_3dm.json")
    o = Oracle(path)
    o.build_preconditioner()
    g = fg.Reconstructor(path, devices=devices)
    lay = smooth_layers(o, 11)
    for k in range(4):
        s = noisy_slopes(o, lay, 700 + k, o.get_state()["a_prev2"])
        c_o, a_o, rho_o = o.step(s)
        a = g.step(s)
        assert rel_err(g.coeffs(), c_o) <= 1e-9, ("c", k)
        assert rel_err(a, a_o) <= 1e-9, ("a", k)
        assert rel_err(g.last_rho, rho_o) <= 1e-9, ("rho", k)
    st = o.get_state()
    g.reset()
    g.set_state(st)  # every shard restarts from the oracle's state
    s = noisy_slopes(o, lay, 800, st["a_prev2"])
    c_o, a_o, _ = o.step(s)
    assert rel_err(g.step(s), a_o) <= 1e-10
