"""The reference-side C++ drop-in (include/fewha_gpu_reconstructor.hpp) driven by
the reference's own caller loops (tests/cpp/test_dropin.cpp): run_bench's closed
loop (bench.hpp:144-154), run_closed_loop with evaluate_quality
(simulation.hpp:321-345), the full ReconstructorState mirror, reset and the
exception mapping -- GPU wrapper vs the unmodified fewha::Reconstructor, compiled
together from the reference headers in place (tests/cpp/Makefile)."""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
BIN = os.path.join(ROOT, "tests", "cpp", "_build", "test_dropin")


@pytest.mark.skipif(not os.path.exists(BIN), reason="tests/cpp/_build/test_dropin not built (needs /root/reference)")
def test_reference_callers_through_the_cpp_dropin():
    out = subprocess.run([BIN, os.path.join(ROOT, "presets")], capture_output=True, text=True, timeout=900)
    print(out.stdout[-4000:], out.stderr[-2000:])
    assert out.returncode == 0, out.stdout[-4000:] + out.stderr[-2000:]
    assert "PASSED" in out.stdout
