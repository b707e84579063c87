"""The drop-in boundary, checked without a GPU.

* librlra_b200.so loads and exports every function include/rlra_c.h
  declares (the C-ABI a reference-side binding links against);
* the host RNG the product uses for parity-mode Omega is the reference's
  stream bit for bit (golden vectors from the reference);
* with no usable device, the engine refuses loudly (no CPU fallback);
* the C++ drop-in headers (include/rlra/*.hpp) compile against the C-ABI.
"""
import os
import re
import shutil
import subprocess

import numpy as np
import pytest

import paper_1502_05366_b200 as R

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rlra_c.h")
GOLD = os.path.join(ROOT, "tests", "golden", "golden.npz")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = set(re.findall(r"\b(rlra_[a-z0-9_]+)\s*\(", src))
    return sorted(n for n in names if not n.endswith("_fn"))


def test_library_exports_every_declared_symbol():
    out = subprocess.run(["nm", "-D", "--defined-only", R.LIB_PATH], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\sT\s(rlra_\w+)", out))
    decl = declared_functions()
    assert len(decl) >= 30
    missing = [d for d in decl if d not in exported]
    assert not missing, missing


def test_library_loads_and_reports_version():
    assert b"sm_100a" in R.lib().rlra_version()


def test_library_is_sm100a_only():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", R.LIB_PATH],
                         capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    arches = set(re.findall(r"sm_(\d+a?)", out.stdout))
    assert arches == {"100a"}, arches


def test_dmma_in_sass():
    """The GEMM kernels are FP64 tensor-core code (SASS DMMA.8x8x4)."""
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", R.LIB_PATH],
                         capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "DMMA.8x8x4" in out.stdout


def test_host_rng_matches_reference_stream():
    g = np.load(GOLD)
    r = R.Rng(12345)
    assert np.array_equal(R.gaussian_matrix(7, 3, r), g["rng_12345_7x3"])
    assert np.array_equal(R.gaussian_matrix(5, 1, r), g["rng_12345_next_5x1"])
    r = R.Rng(42)
    c1, c2 = r.substream(), r.substream()
    assert np.array_equal(R.gaussian_matrix(4, 2, c1), g["rng_42_sub1_4x2"])
    assert np.array_equal(R.gaussian_matrix(4, 2, c2), g["rng_42_sub2_4x2"])


def test_host_rng_matches_oracle_long_stream(orc):
    r = R.Rng(987)
    o = orc.rng(987)
    assert np.array_equal(R.gaussian_matrix(333, 7, r), orc.gaussian(333, 7, o))
    assert r.state()[0] == tuple(o.s)


def _have_gpu():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_have_gpu(), reason="checks the no-device path")
def test_no_device_fails_loudly():
    with pytest.raises(R.RlraError):
        R.Engine(0)


def test_cpp_dropin_headers_compile(tmp_path):
    if not shutil.which("g++"):
        pytest.skip("no g++")
    src = tmp_path / "t.cpp"
    src.write_text(
        '#include "rlra/rlra.hpp"\n#include "rlra/io.hpp"\n#include "rlra/testmat.hpp"\n'
        '#include "rlra/report.hpp"\n#include "rlra/rsvd.hpp"\n#include "rlra/interp.hpp"\n'
        'int main(){ rlra::RngState r(1);\n'
        '  rlra::TestMatrix t = rlra::gen_test_matrix(40, 30, rlra::SpectrumSpec::type_ii(), r);\n'
        '  rlra::SvdFactors f = rlra::rsvd_v2(t.a, 5, 5, 1, 1, r);\n'
        '  rlra::ErrorReport e = rlra::verify(t.a, f, t.sigma_true);\n'
        '  rlra::save_binary("x.bin", t.a); rlra::DenseMatrix b = rlra::load_binary("x.bin");\n'
        '  rlra::CurFactors c = rlra::cur_rand(b, 3, 2, 1, 1, r);\n'
        '  (void)e; (void)c; return 0; }\n')
    res = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-I", os.path.join(ROOT, "include"),
                          str(src)], capture_output=True, text=True)
    assert res.returncode == 0, res.stderr


def test_reference_cli_compiles_against_dropin_headers(tmp_path):
    """The reference's UNMODIFIED command-line driver compiles against the
    drop-in headers (include/rlra) with the self-written CLI11 subset
    (tools/cli11) — the source-level drop-in check."""
    src = "/root/reference/proj/tools/rlra_cli.cpp"
    if not os.path.exists(src) or not shutil.which("g++"):
        pytest.skip("reference source or g++ absent")
    res = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-I", os.path.join(ROOT, "include"), "-I",
                          os.path.join(ROOT, "tools", "cli11"), src], capture_output=True, text=True)
    assert res.returncode == 0, res.stderr[-3000:]
