"""Frozen-set files in the reference format (code.cpp:164-194):
files written by either side load identically on the other, and malformed
files fail with the reference's exact messages."""
import numpy as np
import pytest


@pytest.fixture(scope="module")
def P(native):
    import paper_1710_08314_b200 as P

    return P


def test_round_trip_and_cross_load(P, ref_lib, tmp_path):
    rng = np.random.default_rng(5)
    for n in (2, 64, 2048):
        k = int(rng.integers(1, n + 1))
        fz = (rng.random(n) < 0.5).astype(np.uint8)
        a, b = tmp_path / f"ours_{n}.txt", tmp_path / f"ref_{n}.txt"
        P.save_frozen_file(a, n, k, fz)
        ref_lib.ref_frozen_save(b, n, k, fz)
        assert a.read_bytes() == b.read_bytes()
        for path in (a, b):
            n2, k2, m2 = P.load_frozen_file(path)
            rn, rk, rm = ref_lib.ref_frozen_load(path)
            assert (n2, k2) == (n, k) == (rn, rk)
            assert np.array_equal(m2, fz) and np.array_equal(rm, fz)


@pytest.mark.parametrize("text", ["", "8", "x 4\n00001111\n", "8 4\n", "8 4\n0000111\n",
                                  "8 4\n0000111x\n", "4 2 0110\n"])
def test_malformed_files_match_reference(P, ref_lib, tmp_path, text):
    path = tmp_path / "f.txt"
    path.write_text(text)
    try:
        ref = ref_lib.ref_frozen_load(path)
        ref_err = None
    except RuntimeError as e:
        ref, ref_err = None, e.args
    if ref_err is None:
        n, k, m = P.load_frozen_file(path)
        assert (n, k) == ref[:2] and np.array_equal(m, ref[2])
    else:
        with pytest.raises(P.ParseError) as ei:
            P.load_frozen_file(path)
        assert ref_err[0] == "parse" and str(ei.value) == ref_err[1]


def test_missing_file_is_io_error(P, tmp_path):
    with pytest.raises(P.IoError) as ei:
        P.load_frozen_file(tmp_path / "none.txt")
    assert "cannot open" in str(ei.value)
