"""Binary matrix I/O to device row shards, the test-matrix generator and the
SVD verifier (csrc/io.cu) against the unmodified reference (oracle/_ref):
bit-exact round trips with files the reference writes, the reference's
non-finite message, the generator's exact spectrum, and verify()'s numbers."""
import ctypes as C
import os

import numpy as np
import pytest

import _oracle
import paper_1502_05366_b200 as R

pytestmark = pytest.mark.gpu


def _ref():
    if not os.path.exists(_oracle.REF_PATH):
        pytest.skip("oracle/_ref not built")
    lib = C.CDLL(_oracle.REF_PATH)
    lib.ref_last_error.restype = C.c_char_p
    return lib


def test_binary_round_trip_and_reference_files(eng, tmp_path):
    lib = _ref()
    rs = np.random.default_rng(1)
    a = np.asfortranarray(rs.standard_normal((1031, 77)))
    p_ref = str(tmp_path / "ref.bin")
    assert lib.ref_save_binary(os.fsencode(p_ref), _oracle.d(a), 1031, 77) == 0
    # the reference's file, loaded whole and as row shards, bit for bit
    np.testing.assert_array_equal(eng.load_binary(p_ref), a)
    np.testing.assert_array_equal(eng.load_binary(p_ref, 500, 300), a[500:800])
    # our file is byte-identical to the reference's
    p_ours = str(tmp_path / "ours.bin")
    eng.save_binary(p_ours, a)
    assert open(p_ours, "rb").read() == open(p_ref, "rb").read()


def test_binary_load_to_device_shards(eng, tmp_path):
    import torch

    rs = np.random.default_rng(2)
    a = np.asfortranarray(rs.standard_normal((4000, 513)))
    p = str(tmp_path / "a.bin")
    eng.save_binary(p, a)
    bounds = [0, 1333, 2999, 4000]
    for r0, r1 in zip(bounds[:-1], bounds[1:]):
        buf = torch.empty((r1 - r0) * 513, dtype=torch.float64, device="cuda")
        eng.device_load_binary(p, r0, r1 - r0, buf.data_ptr(), r1 - r0)
        got = buf.view(513, r1 - r0).t().cpu().numpy()
        np.testing.assert_array_equal(got, a[r0:r1])


def test_binary_non_finite_value_message_matches_reference(eng, tmp_path):
    lib = _ref()
    a = np.asfortranarray(np.ones((50, 9)))
    a[37, 4] = np.inf
    a[41, 2] = np.nan
    p = str(tmp_path / "bad.bin")
    eng.save_binary(p, a)
    r, c = C.c_int(0), C.c_int(0)
    assert lib.ref_load_binary(os.fsencode(p), C.byref(r), C.byref(c), None) != 0
    want = lib.ref_last_error().decode()
    with pytest.raises(R.IoError) as e:
        eng.load_binary(p)
    assert str(e.value) == want


def test_gen_test_matrix_has_the_requested_spectrum(eng):
    sig = np.exp(-np.arange(60) / 10.0)
    a = eng.gen_test_matrix(400, 250, sig, seed=7)
    s = np.linalg.svd(a, compute_uv=False)
    assert np.max(np.abs(s[:60] - sig) / sig) <= 1e-12
    assert np.max(s[60:]) <= 1e-14
    b = eng.gen_test_matrix(400, 250, sig, seed=7, noise=1e-3)
    assert 0.5e-3 < np.linalg.norm(b - a) / np.sqrt(400 * 250) < 2e-3
    np.testing.assert_array_equal(eng.gen_test_matrix(400, 250, sig, seed=7), a)  # deterministic


def test_verify_svd_matches_reference(eng):
    lib = _ref()
    sig = np.exp(-np.arange(120) / 15.0)
    a = eng.gen_test_matrix(300, 200, sig, seed=3)
    u, s, v = eng.rsvd_v2(a, 20, 5, 1, 1, rng=R.Rng(9))
    got = eng.verify_svd(a, u, s, v, sig)
    out = np.zeros(5)
    uf, vf = np.asfortranarray(u), np.asfortranarray(v)
    assert lib.ref_verify_svd(_oracle.d(np.asfortranarray(a)), 300, 200, _oracle.d(uf), _oracle.d(np.ascontiguousarray(s)),
                              _oracle.d(vf), 20, _oracle.d(np.ascontiguousarray(sig)), 120, _oracle.d(out)) == 0
    assert abs(got["rel_frobenius_error"] - out[0]) <= 1e-10 * out[0]
    assert abs(got["rel_spectral_error"] - out[1]) <= 1e-8 * out[1]
    np.testing.assert_allclose([got["fro_floor"], got["spec_floor"], got["spec_bound"]], out[2:], rtol=1e-14)
