"""Binary matrix file validation (reference io.hpp:66-109), CPU only: the
header check of librlra_b200 (rlra_binary_header, no device needed) raises
IoError with the reference's own message for every malformed file, compared
against the unmodified reference's load_binary where oracle/_ref is built."""
import ctypes as C
import os
import struct

import numpy as np
import pytest

import _oracle
import paper_1502_05366_b200 as R


def _ref_message(path):
    if not os.path.exists(_oracle.REF_PATH):
        return None
    lib = C.CDLL(_oracle.REF_PATH)
    lib.ref_last_error.restype = C.c_char_p
    r, c = C.c_int(0), C.c_int(0)
    st = lib.ref_load_binary(os.fsencode(path), C.byref(r), C.byref(c), None)
    return None if st == 0 else lib.ref_last_error().decode()


def _write(path, data: bytes):
    with open(path, "wb") as f:
        f.write(data)
    return str(path)


def _cases(tmp_path):
    good = struct.pack("<ii", 3, 2) + np.arange(6, dtype="<f8").tobytes()
    return {
        "missing": str(tmp_path / "nope.bin"),
        "short_header": _write(tmp_path / "h.bin", b"\x01\x00\x00\x00"),
        "zero_rows": _write(tmp_path / "z.bin", struct.pack("<ii", 0, 5)),
        "negative_cols": _write(tmp_path / "n.bin", struct.pack("<ii", 4, -1)),
        "truncated": _write(tmp_path / "t.bin", good[:-8]),
        "oversized": _write(tmp_path / "o.bin", good + b"\x00"),
    }


@pytest.mark.parametrize("case", ["missing", "short_header", "zero_rows", "negative_cols", "truncated",
                                  "oversized"])
def test_binary_header_rejects_malformed_files_like_the_reference(tmp_path, case):
    path = _cases(tmp_path)[case]
    with pytest.raises(R.IoError) as e:
        R.Engine.binary_header(path)
    want = _ref_message(path)
    if want is not None:
        assert str(e.value) == want
    assert "load_binary: " in str(e.value)


def test_binary_header_reads_dimensions(tmp_path):
    data = struct.pack("<ii", 3, 2) + np.arange(6, dtype="<f8").tobytes()
    assert R.Engine.binary_header(_write(tmp_path / "g.bin", data)) == (3, 2)
