"""The C++ drop-in end to end: a reference-style program using only the
rlra:: API is compiled against include/rlra, linked with librlra_b200.so and
run on the GPU."""
import os
import shutil
import subprocess

import pytest

import paper_1502_05366_b200 as R

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_dropin_program_runs_on_the_engine(tmp_path):
    if not shutil.which("g++"):
        pytest.skip("no g++")
    libdir = os.path.dirname(R.LIB_PATH)
    exe = tmp_path / "dropin"
    build = subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"),
                            os.path.join(ROOT, "tests", "cpp", "dropin_demo.cpp"), "-L", libdir, "-lrlra_b200",
                            f"-Wl,-rpath,{libdir}", "-o", str(exe)], capture_output=True, text=True)
    assert build.returncode == 0, build.stderr
    run = subprocess.run([str(exe), str(tmp_path / "a.bin")], capture_output=True, text=True, timeout=300)
    assert run.returncode == 0, (run.returncode, run.stdout, run.stderr)
    assert "dropin ok" in run.stdout
