"""The C oracle (oracle/polar_oracle.c) pinned before it is trusted:
  * against the golden vectors the UNMODIFIED reference produced
    (tests/golden/make_golden.py), bit for bit: payload, codeword, crc_ok,
    escalation level and metric for every decoder kind and precision;
  * against the reference's own pinned unit-test values
    (test_kernels.cpp, test_select.cpp, test_list.cpp, test_bits_crc.cpp);
  * against the compiled reference itself on fresh seeded inputs, when
    oracle/_ref is available.
"""
import ctypes as C
import glob
import os

import numpy as np
import pytest

from conftest import rough_llrs

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CRC_SPECS = {
    "32-GZIP": (32, 0x04C11DB7, 1, 0xFFFFFFFF, 0xFFFFFFFF),
    "16-CCITT": (16, 0x1021, 0, 0xFFFF, 0),
    "8": (8, 0x07, 0, 0, 0),
    "11:621:0:0:0": (11, 0x621, 0, 0, 0),
    "24:b2b117:0:0:0": (24, 0xB2B117, 0, 0, 0),
}


def _orc(oracle_lib, n, k, fz, crc, kind, l, prec, pr):
    return oracle_lib.Oracle(n, k, fz, CRC_SPECS[crc] if crc else None, kind, l, prec, pr)


def decode_fixtures():
    return sorted(glob.glob(os.path.join(GOLD, "decode_*.npz")))


@pytest.mark.parametrize("path", decode_fixtures(), ids=lambda p: os.path.basename(p)[7:-4])
def test_oracle_matches_reference_golden(oracle_lib, path):
    z = np.load(path, allow_pickle=False)
    n, k, crc = int(z["n"]), int(z["k"]), str(z["crc"])
    pr = tuple(int(x) for x in z["pruning"])
    for j in range(int(z["runs"])):
        kind, l = str(z[f"r{j}_kind"]), int(z[f"r{j}_l"])
        o = _orc(oracle_lib, n, k, z["frozen"], crc, kind, l, str(z["precision"]), pr).decode(z["llr"])
        tag = f"{os.path.basename(path)} {kind} L={l}"
        assert np.array_equal(o.payload, z[f"r{j}_payload"]), tag
        assert np.array_equal(o.codeword, z[f"r{j}_codeword"]), tag
        assert np.array_equal(o.crc_ok, z[f"r{j}_crc_ok"]), tag
        assert np.array_equal(o.esc, z[f"r{j}_esc"]), tag
        assert np.array_equal(o.metric, z[f"r{j}_metric"]), tag


def test_oracle_crc_golden(oracle_lib):
    z = np.load(os.path.join(GOLD, "crc.npz"))
    msg = np.unpackbits(np.frombuffer(b"123456789", np.uint8))
    i = 0
    while f"check_{i}_spec" in z:
        spec = tuple(int(x) for x in z[f"check_{i}_spec"])
        assert oracle_lib.oracle_crc(spec, msg) == int(z[f"check_{i}_value"])
        bits, off = z[f"rand_{i}_bits"], 0
        for L, want in zip(z[f"rand_{i}_lens"], z[f"rand_{i}_crc"]):
            assert oracle_lib.oracle_crc(spec, bits[off:off + L]) == int(want)
            off += L
        i += 1
    assert i >= 5


def test_crc_published_check_values(oracle_lib):
    """test_bits_crc.cpp:119-128: '123456789' -> 0xCBF43926 / 0x29B1 / 0xF4."""
    msg = np.unpackbits(np.frombuffer(b"123456789", np.uint8))
    assert oracle_lib.oracle_crc(CRC_SPECS["32-GZIP"], msg) == 0xCBF43926
    assert oracle_lib.oracle_crc(CRC_SPECS["16-CCITT"], msg) == 0x29B1
    assert oracle_lib.oracle_crc(CRC_SPECS["8"], msg) == 0xF4
    assert oracle_lib.oracle_crc(CRC_SPECS["32-GZIP"], np.zeros(0, np.uint8)) == 0


def test_oracle_tree_golden(oracle_lib):
    z = np.load(os.path.join(GOLD, "trees.npz"))
    for i in range(int(z["count"])):
        got = oracle_lib.oracle_tree(z[f"t{i}_frozen"], tuple(int(x) for x in z[f"t{i}_cfg"]))
        assert np.array_equal(got, z[f"t{i}_nodes"]), i


def _kern(oracle_lib, prec):
    lib = C.CDLL(oracle_lib.build_oracle())
    if prec == "f32":
        lib.orc_kernels_f32.argtypes = [C.c_float, C.c_float, C.c_void_p]

        def k(a, b):
            out = np.zeros(5, np.float32)
            lib.orc_kernels_f32(a, b, out.ctypes.data_as(C.c_void_p))
            return out
    else:
        lib.orc_kernels_i8.argtypes = [C.c_int, C.c_int, C.c_void_p]

        def k(a, b):
            out = np.zeros(5, np.int32)
            lib.orc_kernels_i8(a, b, out.ctypes.data_as(C.c_void_p))
            return out
    return k


def test_pinned_kernel_values(oracle_lib):
    """test_kernels.cpp:11-37 pinned f / g / sat / hard values."""
    kf, k8 = _kern(oracle_lib, "f32"), _kern(oracle_lib, "i8")
    assert kf(2.0, -3.0)[0] == -2.0
    assert kf(0.0, 5.0)[0] == 0.0
    assert kf(-4.0, -4.0)[0] == 4.0
    assert k8(2, -3)[0] == -2 and k8(0, -5)[0] == 0
    assert kf(2.0, 3.0)[1] == 5.0 and kf(2.0, 3.0)[2] == 1.0
    assert k8(100, 100)[1] == 127
    assert k8(-100, 100)[2] == 127
    assert k8(100, -100)[2] == -127
    assert k8(120, 120)[3] == 127 and k8(-120, -120)[3] == -127
    assert kf(0.0, 0.0)[4] == 0 and k8(0, 0)[4] == 0
    assert kf(-0.5, 0.0)[4] == 1


def test_two_smallest_matches_naive(oracle_lib):
    """test_select.cpp:57-72: two smallest under (value, index), heavy ties."""
    lib = C.CDLL(oracle_lib.build_oracle())
    lib.orc_two_smallest_f32.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
    rng = np.random.default_rng(31)
    for n in list(range(2, 41)) + [81, 163, 327, 655]:
        for _ in range(10):
            v = rng.integers(0, 7, n).astype(np.float32)
            i1, i2 = C.c_int(), C.c_int()
            lib.orc_two_smallest_f32(v.ctypes.data_as(C.c_void_p), n, C.byref(i1), C.byref(i2))
            order = sorted(range(n), key=lambda i: (v[i], i))
            assert (i1.value, i2.value) == (order[0], order[1])


def _bits(s):
    return np.array([c == "1" for c in s], np.uint8)


NONE = (0, 0, 0, 0, 0, 0)
DEFAULT = (1, 1, 1, 1, 0, 4)


def test_pinned_list_penalties(oracle_lib):
    """test_list.cpp:78-193: single-node penalties, forks and the four-way tie."""
    O = oracle_lib.Oracle
    # frozen leaf: penalty is the disagreeing magnitude
    d = O(2, 1, _bits("10"), None, "scl", 1, "f32", NONE)
    p, cw, ok, met, alive, sm = d.list_decode(np.array([-2, 5], np.float32), 1, False)
    assert met == 2.0 and np.unpackbits(cw)[:2].tolist() == [0, 0]
    # info leaf fork
    d = O(2, 1, _bits("01"), None, "scl", 2, "f32", NONE)
    p, cw, ok, met, alive, sm = d.list_decode(np.array([3, 3], np.float32), 2, False)
    assert met == 0.0 and np.unpackbits(p)[0] == 0 and alive.sum() == 2 and sm.max() == 3.0
    # rate-0 subtree sums every negative magnitude
    d = O(8, 4, _bits("11110000"), None, "sscl", 1, "f32", DEFAULT)
    p, cw, ok, met, *_ = d.list_decode(np.array([1, -2, 3, -4, 100, 100, 100, 100], np.float32), 1, False)
    assert met == 6.0
    # repetition fork: all-one beats all-zero
    d = O(4, 1, _bits("1110"), None, "sscl", 2, "f32", DEFAULT)
    p, cw, ok, met, alive, sm = d.list_decode(np.array([1, 1, 1, -5], np.float32), 2, False)
    assert met == 3.0 and np.unpackbits(cw)[:4].tolist() == [1, 1, 1, 1] and sm.max() == 5.0
    # rate-1 keeps the hard decision
    d = O(4, 4, _bits("0000"), None, "sscl", 1, "f32", DEFAULT)
    p, cw, ok, met, *_ = d.list_decode(np.array([9, -8, 1, -2], np.float32), 1, False)
    assert np.unpackbits(cw)[:4].tolist() == [0, 1, 0, 1] and met == 0.0
    # SPC, parity intact / broken
    d = O(4, 3, _bits("1000"), None, "sscl", 2, "f32", DEFAULT)
    p, cw, ok, met, alive, sm = d.list_decode(np.array([1, 5, -6, -7], np.float32), 2, False)
    assert np.unpackbits(cw)[:4].tolist() == [0, 0, 1, 1] and met == 0.0 and sm.max() == 6.0
    p, cw, ok, met, alive, sm = d.list_decode(np.array([1, 5, -6, 7], np.float32), 2, False)
    assert np.unpackbits(cw)[:4].tolist() == [1, 0, 1, 0] and met == 1.0 and sm.max() == 5.0
    # four-way tie keeps the earliest candidates
    d = O(2, 2, _bits("00"), None, "scl", 2, "f32", NONE)
    p, cw, ok, met, alive, sm = d.list_decode(np.array([0, 0], np.float32), 2, False)
    assert met == 0.0 and np.unpackbits(p)[:2].tolist() == [0, 0] and alive.sum() == 2
    assert sm[0] == 0.0 and sm[1] == 0.0


def test_fixed_point_metrics_normalised(oracle_lib):
    """test_list.cpp:321-356: int8 metrics in [0, 127], min alive metric 0."""
    from oracle.oracle import ref_construct_frozen, Reference  # noqa: F401
    rng = np.random.default_rng(404)
    fz = np.zeros(64, np.uint8)
    fz[np.argsort(rng.random(64))[:32]] = 1
    d = oracle_lib.Oracle(64, 32, fz, None, "sscl", 8, "i8", DEFAULT)
    for _ in range(50):
        mag = np.where(rng.integers(0, 3, 64) > 0, 127, rng.integers(0, 8, 64))
        v = (np.where(rng.integers(0, 2, 64) == 1, -1, 1) * mag).astype(np.int8)
        *_, alive, sm = d.list_decode(v, 8, False)
        live = sm[alive == 1]
        assert live.min() == 0 and live.max() <= 127 and live.min() >= 0


def test_oracle_config_errors(oracle_lib):
    """test_list.cpp:509-539: bad list sizes and missing CRCs are rejected."""
    O = oracle_lib.Oracle
    fz = _bits("1111000011110000")
    with pytest.raises(ValueError):
        O(16, 8, fz, None, "scl", 3, "f32", NONE)
    with pytest.raises(ValueError):
        O(16, 8, fz, None, "ca_sscl", 4, "f32", DEFAULT)
    fz12 = _bits("1111000000000000")
    O(16, 4, fz12, CRC_SPECS["8"], "pa_sscl", 2, "f32", DEFAULT)  # valid
    with pytest.raises(ValueError):
        O(16, 4, fz12, CRC_SPECS["8"], "pa_sscl", 1, "f32", DEFAULT)  # adaptive needs L >= 2
    with pytest.raises(ValueError):
        O(16, 4, fz12, CRC_SPECS["8"], "sscl", 6, "f32", DEFAULT)  # not a power of two
    with pytest.raises(ValueError):
        O(16, 7, fz, None, "sc", 1, "f32", NONE)  # 8 open positions != K


@pytest.mark.parametrize("prec", ["f32", "i8"])
def test_oracle_vs_compiled_reference_fresh(oracle_lib, prec):
    """Fresh seeded inputs through both CPU implementations (skipped where
    oracle/_ref could not be built)."""
    from oracle import oracle as O
    try:
        O.Reference.lib()
    except Exception as e:  # noqa: BLE001
        pytest.skip(f"reference not available: {e}")
    rng = np.random.default_rng(77 + (prec == "i8"))
    for n, k, crc in [(64, 24, "8"), (512, 200, "16-CCITT")]:
        w = CRC_SPECS[crc][0]
        fz = O.ref_construct_frozen(n, k + w, 0.5)
        llr = rough_llrs(rng, n, 32, prec)
        pr = (1, 1, 1, 1, 8, 4) if prec == "i8" else DEFAULT
        for kind, l in [("sc", 1), ("ssc", 1), ("scl", 4), ("sscl", 8), ("ca_sscl", 8),
                        ("pa_sscl", 4), ("fa_sscl", 16)]:
            a = O.Reference(n, k, fz, crc, kind, l, prec, pr).decode(llr)
            b = _orc(oracle_lib, n, k, fz, crc, kind, l, prec, pr).decode(llr)
            for f in ("payload", "codeword", "crc_ok", "esc", "metric"):
                assert np.array_equal(getattr(a, f), getattr(b, f)), (n, kind, l, f)
