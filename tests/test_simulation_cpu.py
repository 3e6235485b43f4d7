"""CPU checks of the simulation harness's host part: the SplitMix64 seed
derivation (simulation.hpp:31-36) the per-frame noise seeds come from.  The
streams, screens, synthesis, quality and loops run on the device and are
pinned to the reference in tests/test_gpu_simulation.py."""
from paper_2009_00946_b200 import simulation as sim


def test_splitmix64_known_answers():
    # SplitMix64 (Steele, Lea, Flood 2014) from state 0 / 1: the first outputs
    assert sim.splitmix64(0) == 0xE220A8397B1DCDAF
    assert sim.splitmix64(1) == 0x910A2DEC89025CC1


def test_splitmix64_wraps_mod_2_64():
    assert sim.splitmix64((1 << 64) + 5) == sim.splitmix64(5)  # seeds are taken mod 2^64
    assert 0 <= sim.splitmix64((1 << 64) - 1) < (1 << 64)
