"""Matrix files (reference io.cpp:37-121): the library's
writer produces byte-identical files to the reference's writer, and each side
reads what the other wrote -- both formats, edge shapes (empty, 1 x 1,
non-square), special values; malformed files raise like the reference."""
import os

import numpy as np
import pytest


CASES = [np.zeros((0, 0)), np.array([[5.0]]), np.arange(6.0).reshape(2, 3) - 2.5,
         np.array([[1e-300, -0.0, np.pi], [1e300, 2.0 ** -1074, -1.0 / 3.0]]),
         np.random.default_rng(3).standard_normal((17, 9))]


@pytest.mark.parametrize("fmt", ["teig", "matrixmarket"])
@pytest.mark.parametrize("k", range(len(CASES)))
def test_round_trip_and_bytes_match_reference(T, O, tmp_path, fmt, k):
    from paper_2002_05024_b200 import io
    a = CASES[k]
    ours = os.path.join(tmp_path, "ours." + fmt)
    io.write_matrix_file(ours, a, fmt)
    b = io.read_matrix_file(ours, fmt)
    assert b.shape == a.shape and np.array_equal(b, a)  # exact: 17 digits round-trip doubles
    if os.path.exists(O.REF_IO_TOOL):
        # the reference converts our file to TEIG and back to this format: it
        # reads what we wrote, and its writer produces our bytes
        via = os.path.join(tmp_path, "via.teig")
        theirs = os.path.join(tmp_path, "ref." + fmt)
        O.ref_io_convert(fmt, ours, "teig", via)
        assert np.array_equal(io.read_matrix_file(via, "teig"), a)
        O.ref_io_convert("teig", via, fmt, theirs)
        assert open(ours, "rb").read() == open(theirs, "rb").read()


def test_malformed_files_raise(T, tmp_path):
    from paper_2002_05024_b200 import io
    p = os.path.join(tmp_path, "bad")
    open(p, "wb").write(b"NOPE")
    with pytest.raises(T.TaskeigError):
        io.read_matrix_file(p, "teig")
    open(p, "wb").write(b"TEIG\x02\x00\x00\x00")
    with pytest.raises(T.TaskeigError, match="version"):
        io.read_matrix_file(p, "teig")
    io.write_matrix_file(p, np.ones((4, 4)), "teig")
    open(p, "r+b").truncate(40)
    with pytest.raises(T.TaskeigError, match="truncated"):
        io.read_matrix_file(p, "teig")
    open(p, "w").write("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1.0\n")
    with pytest.raises(T.TaskeigError, match="flavor"):
        io.read_matrix_file(p, "matrixmarket")
    with pytest.raises(T.TaskeigError, match="format"):
        io.write_matrix_file(p, np.ones((2, 2)), "csv")
