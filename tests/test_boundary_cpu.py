"""CPU tests of the drop-in boundary (no GPU needed, no compute calls).

* the sm_100a library loads and exports every symbol include/fewha_gpu.h declares;
* the host-side preset derivation (fewha_gpu_preset_info) reproduces the
  reference's finalize_geometry bitwise (extents, active masks);
* invalid presets are rejected with the reference's error class and message
  (config_error -> FEWHA_CONFIG, geometry.hpp:281-362, config_io.hpp:36-195);
* constructing a Reconstructor without a device fails loudly (no CPU fallback).
"""
import json
import os
import re

import numpy as np
import pytest

import paper_2009_00946_b200 as fg
from conftest import ROOT, preset
from oracle import Oracle, OracleError, RefOracle

HEADER = os.path.join(ROOT, "include", "fewha_gpu.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(fewha_gpu_[a-zA-Z_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = fg.lib()
    syms = declared_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(fg.EXPORTS)


def test_library_is_sm100a():
    """The shipped object carries sm_100a SASS only (cuobjdump -lelf)."""
    import shutil
    import subprocess
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([exe, "-lelf", fg.LIB_PATH], capture_output=True, text=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


@pytest.mark.parametrize("name", ["mini", "small_mcao", "elt_mcao84", "maory9", "small_mcao_2dm", "elt_ltao84",
                                  "elt_mcao84_3dm", "elt_moao84"])
def test_host_geometry_matches_oracle_bitwise(name):
    dims, ext, dext, masks = fg.preset_info(preset(name + ".json"))
    o = Oracle(preset(name + ".json"))
    eo, do_, mo = o.geometry()
    assert dims.n == o.dims.n and dims.S == o.dims.S and dims.A == o.dims.A and dims.Nw == o.dims.Nw
    assert np.array_equal(ext, eo)
    assert np.array_equal(dext, do_)
    assert np.array_equal(masks, mo)


def test_host_geometry_matches_golden_elt():
    g = np.load(os.path.join(ROOT, "tests", "golden", "elt_mcao84_geometry.npz"))
    _, ext, dext, masks = fg.preset_info(preset("elt_mcao84.json"))
    assert np.array_equal(ext, g["layer_extent"]) and np.array_equal(masks, g["masks"])


def _mutations():
    base = json.load(open(preset("small_mcao.json")))
    cases = {}

    def mut(name, fn):
        j = json.loads(json.dumps(base))
        fn(j)
        cases[name] = j

    mut("l_ne_m", lambda j: j["dms"].pop())
    mut("neg_diameter", lambda j: j["telescope"].__setitem__("diameter", -1.0))
    mut("star_count", lambda j: j["guide_stars"].pop())
    mut("heights_order", lambda j: j["layers"][1].__setitem__("height", 0.0))
    mut("strength_sum", lambda j: j["layers"][0].__setitem__("relative_strength", 0.5))
    mut("lgs_low", lambda j: j["guide_stars"][0].__setitem__("height", 5000.0))
    mut("gain", lambda j: j["loop"].__setitem__("gain", 1.5))
    mut("alpha", lambda j: j["solver"].__setitem__("alpha", 0.0))
    mut("order", lambda j: j["solver"].__setitem__("wavelet_order", 11))
    mut("fault", lambda j: j["solver"].__setitem__("fault", "bogus"))
    mut("missing_key", lambda j: j["wfs"][0].pop("n_subap"))
    mut("bad_kind", lambda j: j["guide_stars"][0].__setitem__("kind", "xgs"))
    mut("bad_precond", lambda j: j["solver"].__setitem__("preconditioner", "nope"))
    mut("bad_loop", lambda j: j["loop"].__setitem__("mode", "half"))
    mut("small_extent", lambda j: j["layers"][2].__setitem__("extent", 1.0))
    mut("n_act", lambda j: j["dms"][0].__setitem__("n_act", 1))
    return cases


MUTATIONS = _mutations()


@pytest.mark.parametrize("case", sorted(MUTATIONS))
def test_config_errors_match_reference(case, tmp_path):
    path = tmp_path / f"{case}.json"
    path.write_text(json.dumps(MUTATIONS[case]))
    with pytest.raises(fg.ConfigError) as ei:
        fg.preset_info(path)
    msg = str(ei.value)
    if RefOracle.available():
        with pytest.raises(OracleError) as er:
            RefOracle(path)
        assert er.value.code == 2
        assert msg == str(er.value)
    else:
        assert msg.startswith("invalid geometry:") or msg.startswith("config:")


def test_missing_file_is_config_error(tmp_path):
    with pytest.raises(fg.ConfigError, match="cannot open"):
        fg.preset_info(tmp_path / "nope.json")


def test_malformed_json_is_config_error(tmp_path):
    p = tmp_path / "bad.json"
    p.write_text("{ not json")
    with pytest.raises(fg.ConfigError, match="parse error"):
        fg.preset_info(p)


def test_no_silent_cpu_fallback():
    """Without a CUDA device the product must fail loudly, never compute on the CPU."""
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    with pytest.raises(fg.FewhaError, match="CUDA"):
        fg.Reconstructor(preset("mini.json"))


def test_bench_models_cover_every_kernel_kind():
    """bench.py's algorithmic-bytes model has an entry for every kernel kind the
    library's profile reports (the roofline object must never miss a kind), and the
    frame model matches SURVEY 8(d)'s 71.76 MB at the ELT MCAO-84 scale."""
    import importlib.util

    import paper_2009_00946_b200 as fg

    spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    d = bench.preset_dims(os.path.join(ROOT, "presets", "elt_mcao84_3dm.json"))
    for kind in fg.Reconstructor.KERNEL_KINDS:
        assert bench.kernel_bytes(kind, d, 8) > 0, kind
    assert abs(bench.frame_bytes(d, 8) - 71.76e6) / 71.76e6 < 1e-3


def test_bench_roofline_names_the_dominant_function():
    """The roofline object sums a kernel function's launch kinds (k_inv_cluster =
    inv_pcg0 + inv_pcg + inv_fit) before taking the largest share, and every kind
    maps to a kernel function."""
    import importlib.util

    import paper_2009_00946_b200 as fg

    spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    for kind in fg.Reconstructor.KERNEL_KINDS:
        assert kind in bench.FUNC, kind
    prof = {"k_inv_cluster": {"share": 0.31, "achieved_gbs": 578.0, "bytes_per_launch": 1.1e7, "launch_ms": 0.019,
                              "launches_per_frame": 5},
            "k_gather": {"share": 0.21, "achieved_gbs": 116.0, "bytes_per_launch": 1.5e6, "launch_ms": 0.013,
                         "launches_per_frame": 5}}
    r = bench.roofline_object(prof, 6548.2, "measured", "fp64", "test")
    assert r["kernel"] == "k_inv_cluster" and abs(r["frac"] - 578.0 / 6548.2) < 1e-4


@pytest.mark.skipif(not os.path.isdir("/root/reference/proj/include"), reason="reference headers absent")
def test_cpp_dropin_builds_against_the_reference_headers():
    """include/fewha_gpu_reconstructor.hpp compiles against the unmodified reference
    headers and links the in-tree library (tests/cpp/Makefile); the GPU test runs it."""
    import subprocess

    out = subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    binp = os.path.join(ROOT, "tests", "cpp", "_build", "test_dropin")
    ldd = subprocess.run(["ldd", binp], capture_output=True, text=True).stdout
    assert "libfewha_gpu.so" in ldd and "not found" not in ldd.split("libfewha_gpu.so")[1].splitlines()[0]
