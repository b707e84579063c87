"""The reference's own command-line driver (tools/rlra_cli.cpp, unmodified)
compiled against the drop-in headers (tools/Makefile -> tools/_bin/rlra) and
run on the B200 engine: gen | svd | id | cur | qb | verify | bench with
CSV on stdout (report.hpp:210-244)."""
import csv
import io
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "tools", "_bin", "rlra")
HEADER = ("method,m,n,k,params,rel_fro_error,rel_spec_error,fro_floor,spec_floor,spec_bound,nnz_total,seconds")


def run(*args):
    p = subprocess.run([CLI, *args], capture_output=True, text=True, timeout=600)
    return p.returncode, p.stdout, p.stderr


def rows(out):
    lines = out.strip().splitlines()
    assert lines[0] == HEADER
    return list(csv.DictReader(io.StringIO(out)))


@pytest.fixture(scope="module")
def matrix(tmp_path_factory):
    if not os.path.exists(CLI):
        pytest.skip("tools/_bin/rlra not built (needs /root/reference at build time)")
    d = tmp_path_factory.mktemp("cli")
    a = str(d / "a.bin")
    rc, _, err = run("gen", "--m", "300", "--n", "200", "--type", "III", "--seed", "7", "--out", a)
    assert rc == 0, err
    assert os.path.exists(a + ".sigma")
    return d, a


def test_cli_svd_methods_and_verify(matrix):
    d, a = matrix
    for method in ("rand", "blockrand", "det"):
        rc, out, err = run("svd", "--in", a, "--k", "20", "--method", method, "--out-prefix", str(d / method))
        assert rc == 0, err
        r = rows(out)[0]
        assert r["method"] == "svd" and int(r["k"]) == 20
        # randomized and deterministic SVDs sit on the optimal floor
        assert float(r["rel_fro_error"]) <= 1.5 * float(r["fro_floor"])
        rc, out, err = run("verify", "--in", a, "--prefix", str(d / method))
        assert rc == 0, err
        v = rows(out)[0]
        assert abs(float(v["rel_fro_error"]) - float(r["rel_fro_error"])) <= 1e-10
    rc, out, _ = run("svd", "--in", a, "--tol", "1e-3", "--relative", "--method", "blockrand", "--block", "8")
    assert rc == 0 and float(rows(out)[0]["rel_fro_error"]) <= 1e-3


def test_cli_id_cur_qb_and_bench(matrix):
    d, a = matrix
    for cmd, extra in (("id", ["--method", "rand"]), ("cur", ["--method", "rand"]), ("qb", ["--method", "blockrand"]),
                       ("qb", ["--method", "parallel"]), ("qb", ["--method", "hier", "--row-blocks", "2"])):
        rc, out, err = run(cmd, "--in", a, "--k", "16", *extra, "--out-prefix", str(d / cmd))
        assert rc == 0, (cmd, extra, err)
        r = rows(out)[0]
        err_fro, floor = float(r["rel_fro_error"]), float(r["fro_floor"])
        assert r["method"] == cmd and 0.99 * floor <= err_fro <= 1.0
    rc, out, err = run("bench", "--in", a, "--ks", "5,10,20", "--algo", "svd")
    assert rc == 0, err
    b = rows(out)
    assert [int(x["k"]) for x in b] == [5, 10, 20]
    assert float(b[0]["rel_fro_error"]) > float(b[2]["rel_fro_error"])
    # usage errors are the reference's (exit 2)
    rc, _, err = run("svd", "--in", a, "--k", "5", "--tol", "1e-3")
    assert rc == 2 and "exactly one of --k and --tol" in err
