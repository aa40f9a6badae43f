"""Host-side logic of the product library, no GPU needed: the C ABI loads and
exports every declared symbol, CRC parsing/engine, decode-tree construction,
the frame-keyed channel and the create-time validation (ConfigError /
ParseError mapping, decoders.hpp:40-55, code.cpp:82-124, crc.cpp:42-95,
prune_tree.cpp:24-35)."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


@pytest.fixture(scope="module")
def P(native):
    import paper_1710_08314_b200 as P

    return P


def declared_symbols():
    syms = []
    for h in ("polar_b200.h", "polar_b200_sim.h"):
        txt = open(os.path.join(ROOT, "include", h)).read()
        syms += re.findall(r"^(?:const\s+)?\w+\s*\**\s*(pl_\w+)\s*\(", txt, re.M)
    return sorted(set(syms))


def test_library_exports_every_declared_symbol(native):
    syms = declared_symbols()
    assert len(syms) >= 15
    missing = [s for s in syms if not hasattr(native, s)]
    assert not missing, missing
    from paper_1710_08314_b200 import _lib

    assert set(_lib.EXPORTS) == set(syms)


def test_crc_parse_presets_and_raw(P):
    assert P.CrcSpec.parse("32-GZIP") == P.CrcSpec(32, 0x04C11DB7, True, 0xFFFFFFFF, 0xFFFFFFFF)
    assert P.CrcSpec.parse("16-CCITT") == P.CrcSpec(16, 0x1021, False, 0xFFFF, 0)
    assert P.CrcSpec.parse("8") == P.CrcSpec(8, 0x07, False, 0, 0)
    raw = P.CrcSpec.parse("10:233:0:3ff:0")  # test_bits_crc.cpp:208-214
    assert (raw.width, raw.poly, raw.reflect, raw.init, raw.xorout) == (10, 0x233, False, 0x3FF, 0)
    for bad in ("bogus", "16:1021:2:0:0", "16:xyz:0:0:0", "1:2:3", ""):
        with pytest.raises(P.ParseError):
            P.CrcSpec.parse(bad)


def test_crc_engine_config_errors(P):
    """test_bits_crc.cpp:219-221."""
    for spec in (P.CrcSpec(70, 0x7, False, 0, 0), P.CrcSpec(8, 0x107, False, 0, 0),
                 P.CrcSpec(8, 0x06, False, 0, 0)):
        with pytest.raises(P.ConfigError):
            P.crc_compute(spec, np.zeros(8, np.uint8))


def test_crc_engine_golden(P):
    z = np.load(os.path.join(GOLD, "crc.npz"))
    msg = np.unpackbits(np.frombuffer(b"123456789", np.uint8))
    i = 0
    while f"check_{i}_spec" in z:
        w, poly, refl, init, xo = (int(x) for x in z[f"check_{i}_spec"])
        spec = P.CrcSpec(w, poly, bool(refl), init, xo)
        assert P.crc_compute(spec, msg) == int(z[f"check_{i}_value"])
        bits, off = z[f"rand_{i}_bits"], 0
        for L, want in zip(z[f"rand_{i}_lens"], z[f"rand_{i}_crc"]):
            assert P.crc_compute(spec, bits[off:off + L]) == int(want)
            off += L
        i += 1


def test_crc_matches_bit_serial_definition(P):
    """test_bits_crc.cpp:130-165: table engine == bit-serial register for
    widths 3..64, reflected and not, every length class."""
    rng = np.random.default_rng(2024)

    def serial(s, bits):
        mask = (1 << s.width) - 1
        if s.reflect:
            rev = lambda v: int(f"{v:0{s.width}b}"[::-1], 2)
            reg, rp = rev(s.init), rev(s.poly)
            nb = len(bits) // 8
            order = [8 * k + j for k in range(nb) for j in range(7, -1, -1)] + list(range(8 * nb, len(bits)))
            for i in order:
                reg ^= int(bits[i])
                lo = reg & 1
                reg >>= 1
                if lo:
                    reg ^= rp
            return (reg ^ s.xorout) & mask
        reg = s.init & mask
        for b in bits:
            reg ^= int(b) << (s.width - 1)
            top = (reg >> (s.width - 1)) & 1
            reg = (reg << 1) & mask
            if top:
                reg ^= s.poly
        return (reg ^ s.xorout) & mask

    for w in (3, 5, 8, 11, 16, 24, 32, 48, 64):
        for rep in range(4):
            mask = (1 << w) - 1
            s = P.CrcSpec(w, (int(rng.integers(0, 2**62)) | 1) & mask, bool(rep & 1),
                          int(rng.integers(0, 2**62)) & mask, int(rng.integers(0, 2**62)) & mask)
            for L in (0, 1, 5, 7, 8, 9, 15, 16, 17, 40, 63, 64, 65):
                b = rng.integers(0, 2, L).astype(np.uint8)
                assert P.crc_compute(s, b) == serial(s, b), (w, rep, L)


def test_tree_golden(P):
    z = np.load(os.path.join(GOLD, "trees.npz"))
    for i in range(int(z["count"])):
        c = [int(x) for x in z[f"t{i}_cfg"]]
        cfg = P.PruningConfig(bool(c[0]), bool(c[1]), bool(c[2]), bool(c[3]), c[4], c[5])
        assert np.array_equal(P.prune_tree(z[f"t{i}_frozen"], cfg), z[f"t{i}_nodes"]), i


def test_tree_pinned_classifications(P):
    """test_tree.cpp:30-86."""
    b = lambda s: np.array([c == "1" for c in s], np.uint8)
    allc = P.PruningConfig(spc_max=0)
    t = P.prune_tree(b("1100"), allc)
    assert t.shape[0] == 3 and t[t[0, 4], 0] == 3 and t[t[0, 5], 0] == 4
    t = P.prune_tree(b("1110"), allc)
    assert t.shape[0] == 1 and t[0, 0] == 5 and t[0, 3] == 4
    assert P.prune_tree(b("1000"), allc)[0, 0] == 6
    t = P.prune_tree(b("1000"), P.PruningConfig(single_parity=False, spc_max=0))
    assert t[0, 0] == 0 and t[t[0, 4], 0] == 5 and t[t[0, 5], 0] == 4
    assert P.prune_tree(b("10"), allc)[0, 0] == 5  # REP shadows SPC at size 2
    t = P.prune_tree(b("11101000"), P.PruningConfig(rep_max=2, spc_max=4))
    l = t[t[0, 4]]
    assert t[0, 0] == 0 and l[0] == 0 and t[l[4], 0] == 3 and t[l[5], 0] == 5
    assert t[t[0, 5], 0] == 6 and t[t[0, 5], 3] == 4
    for bad in (P.PruningConfig(rep_max=1, spc_max=0), P.PruningConfig(spc_max=2)):
        with pytest.raises(P.ConfigError):
            P.prune_tree(b("1100"), bad)
    with pytest.raises(P.ConfigError):
        P.prune_tree(b("110"), P.PruningConfig())


def test_unpruned_tree_is_full(P):
    fz = P.construct_frozen(64, 32, 0.5)
    t = P.prune_tree(fz, P.PruningConfig.none())
    assert t.shape[0] == 127
    leaves = t[t[:, 0] != 0]
    assert leaves[:, 3].sum() == 64 and (leaves[:, 3] == 1).all()


def test_host_channel_is_the_reference_channel(P):
    """Same (seed, frame) keying, payload, encoder and quantiser as
    run_frame (sim.cpp:48-51): identical info bits and LLR bytes."""
    z = np.load(os.path.join(GOLD, "channel.npz"))
    code = P.make_code(int(z["n"]), int(z["k"]), z["frozen"], str(z["crc"]))
    info, llr = P.channel(code, float(z["ebn0"]), int(z["seed"]), int(z["frame0"]), 8, "f32")
    assert np.array_equal(info, z["info"])
    assert np.array_equal(llr, z["llr"])
    info8, llr8 = P.channel(code, float(z["ebn0"]), int(z["seed"]), int(z["frame0"]), 8, "i8",
                            float(z["scale8"]))
    assert np.array_equal(info8, z["info8"]) and np.array_equal(llr8, z["llr8"])


def test_frame_keyed_channel_matches_range_channel(P):
    """pl_channel_generate_frames with explicit global indices == the range
    form; rows land in a wider batch."""
    code = P.make_code(256, 100, P.construct_frozen(256, 116, 0.5), "16-CCITT")
    info, llr = P.channel(code, 2.0, 5, 40, 12, "f32")
    ids = np.arange(40, 52)[::-1].copy()
    wl = np.zeros((12, 300), np.float32)
    wi = np.zeros((12, 130), np.uint8)
    P.polar.channel_frames(code, 2.0, 5, ids, wl, wi, "f32")
    assert np.array_equal(wl[:, :256], llr[::-1]) and np.array_equal(wi[:, :100], info[::-1])
    assert not wl[:, 256:].any() and not wi[:, 100:].any()


def test_mixed_mcs_workload_codes(P):
    from paper_1710_08314_b200.workload import MixedWorkload

    wl = MixedWorkload()
    codes = wl.code_list()
    assert len(codes) == 31  # (128, 5/6, CRC-24) is infeasible
    assert {c.n for c in codes} == {128, 256, 512, 1024}
    cid = wl.code_ids(0, 100000, 31)
    counts = np.bincount(cid, minlength=31)
    assert counts.min() > 0.8 * 100000 / 31 and np.array_equal(cid, wl.code_ids(0, 100000, 31))


def test_channel_codewords_are_systematic_and_crc_valid(P):
    code = P.make_code(256, 100, P.construct_frozen(256, 116, 0.5), "16-CCITT")
    info, llr = P.channel(code, 30.0, 1, 0, 16, "f32")  # noiseless limit
    x = (llr < 0).astype(np.uint8)
    pay = x[:, code.info_pos]
    assert np.array_equal(pay[:, :100], info)
    for f in range(16):
        assert P.crc_compute(code.crc, pay[f, :100]) == int("".join(map(str, pay[f, 100:])), 2)


def test_frozen_constructions(P):
    fz = P.construct_frozen_ga(2048, 1755, 4.5, 1723 / 2048)
    assert fz.sum() == 2048 - 1755
    fz2 = P.construct_frozen_ga(2048, 1755, 4.5, 1723 / 2048)
    assert np.array_equal(fz, fz2)
    # nested: a lower-rate GA code freezes a superset
    lo = P.construct_frozen_ga(1024, 300, 2.0, 0.3)
    hi = P.construct_frozen_ga(1024, 600, 2.0, 0.3)
    assert (lo >= hi).all()
    b = P.construct_frozen(64, 32, 0.5)
    assert b.sum() == 32 and b[0] == 1 and b[-1] == 0


def test_make_code_validation(P):
    fz = P.construct_frozen(16, 8, 0.5)
    with pytest.raises(P.ConfigError):
        P.make_code(1000, 500, np.zeros(1000))
    with pytest.raises(P.ConfigError):
        P.make_code(16, 0, fz)
    with pytest.raises(P.ConfigError):
        P.make_code(16, 7, fz)
    with pytest.raises(P.ConfigError):
        P.make_code(16, 8, fz, "8")  # 8 open positions, needs 16


def test_decoder_validation_without_gpu(P):
    """FrameDecoder validation (decoders.hpp:40-55) is host-side and raises
    ConfigError before any device work."""
    code = P.make_code(16, 8, P.construct_frozen(16, 8, 0.5))
    crc_code = P.make_code(16, 4, P.construct_frozen(16, 12, 0.5), "8")
    for args in ((code, "ca_sscl", 4), (crc_code, "pa_sscl", 1), (crc_code, "fa_sscl", 1),
                 (crc_code, "sscl", 6), (crc_code, "sscl", 64), (crc_code, "scl", 0)):
        with pytest.raises(P.ConfigError):
            P.FrameDecoder(*args)
    with pytest.raises(P.ConfigError):
        P.FrameDecoder(crc_code, "sscl", 4, pruning=P.PruningConfig(rep_max=1))


def test_no_cpu_fallback(P):
    """A valid decoder on a host without a GPU fails loudly (no fallback)."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("host has a GPU")
    code = P.make_code(16, 8, P.construct_frozen(16, 8, 0.5))
    with pytest.raises(P.DeviceError):
        P.FrameDecoder(code, "sscl", 4)


def test_packed_layout():
    """pack_frames / pack_batch (the pl_decode_packed layout): ascending,
    16-byte aligned offsets, each frame's values in place, both agree."""
    import numpy as np

    from paper_1710_08314_b200.polar import pack_batch, pack_frames

    rng = np.random.default_rng(5)
    for dt in (np.float32, np.int8, np.int16):
        ns = rng.choice([8, 16, 128, 256, 1024], 300)
        llr = rng.integers(-100, 100, (300, 1024)).astype(dt)
        buf, off = pack_frames([llr[f, :ns[f]] for f in range(300)], dt)
        b2, o2 = pack_batch(llr, ns)
        assert np.array_equal(buf, b2) and np.array_equal(off, o2)
        assert (off * np.dtype(dt).itemsize % 16 == 0).all() and (np.diff(off) >= ns[:-1]).all()
        for f in range(300):
            assert np.array_equal(buf[off[f]: off[f] + ns[f]], llr[f, :ns[f]])


def test_interleave32_layout():
    """PL_LLR_INTERLEAVED32 as include/polar_b200.h states it: chunk c (16
    bytes, or the whole frame when shorter) of frame f at chunk index
    ((f // 32) * chunks_per_frame + c) * 32 + f % 32; the last group is
    zero-padded."""
    import numpy as np

    import paper_1710_08314_b200 as P

    rng = np.random.default_rng(0)
    for dt, n, nf in [(np.float32, 64, 70), (np.int8, 64, 33), (np.int16, 8, 5), (np.float32, 2, 40), (np.int8, 8, 64)]:
        x = rng.integers(-100, 100, (nf, n)).astype(dt)
        y = P.interleave32(x).reshape(-1)
        v = min(16 // np.dtype(dt).itemsize, n)
        cpf = n // v
        groups = (nf + 31) // 32
        assert y.size == groups * 32 * n
        for f in range(groups * 32):
            for c in range(cpf):
                at = (((f // 32) * cpf + c) * 32 + f % 32) * v
                want = x[f, c * v:(c + 1) * v] if f < nf else np.zeros(v, dt)
                assert np.array_equal(y[at:at + v], want), (dt, n, f, c)
