"""GPU parity: the sm_100a decoder (through the C ABI) against the C oracle
on identical LLR bytes.  int8 must be bit-exact; float32 is held to the same
exact standard (payload, codeword, crc_ok, escalation level and the float
path metric), which the kernels meet by reproducing the reference's
summation orders and tie rules.
"""
import numpy as np
import pytest

from conftest import rough_llrs

pytestmark = pytest.mark.gpu

KINDS = ["sc", "ssc", "scl", "sscl", "ca_sscl", "pa_sscl", "fa_sscl"]


def _code(P, n, k, crc, design=0.5, ga=None):
    w = P.CrcSpec.parse(crc).width if crc else 0
    if ga is not None:
        fz = P.construct_frozen_ga(n, k + w, ga, k / n)
    else:
        fz = P.construct_frozen(n, k + w, design)
    return P.make_code(n, k, fz, crc)


def _oracle(code, kind, l, prec, pruning):
    from oracle.oracle import Oracle

    crc = code.crc
    spec = (crc.width, crc.poly, int(crc.reflect), crc.init, crc.xorout) if crc else None
    return Oracle(code.n, code.k, code.frozen, spec, kind, l, prec, pruning.as_tuple())


def check_parity(P, torch, code, kind, l, prec, pruning, llr, label=""):
    dec = P.FrameDecoder(code, kind, l, prec, pruning)
    x = torch.from_numpy(np.ascontiguousarray(llr)).cuda()
    out = dec.decode_batch(x, codeword=True)
    torch.cuda.synchronize()
    got = {k: (v.cpu().numpy() if v is not None else None) for k, v in out.items()}
    ref = _oracle(code, kind, l, prec, pruning).decode(llr)
    nf = llr.shape[0]
    pb = (code.payload_size + 7) // 8
    cb = (code.n + 7) // 8
    bad_pay = np.flatnonzero((got["payload"][:, :pb] != ref.payload).any(1))
    bad_cw = np.flatnonzero((got["codeword"][:, :cb] != ref.codeword).any(1))
    bad_ok = np.flatnonzero(got["crc_ok"] != ref.crc_ok)
    bad_esc = np.flatnonzero(got["esc"] != ref.esc)
    bad_met = np.flatnonzero(got["metric"] != ref.metric.astype(np.float32))
    msg = (f"{label} n={code.n} k={code.k} kind={kind} l={l} {prec}: payload {len(bad_pay)}/{nf} "
           f"codeword {len(bad_cw)} crc_ok {len(bad_ok)} esc {len(bad_esc)} metric {len(bad_met)}"
           f" first={[a[:3].tolist() for a in (bad_pay, bad_cw, bad_ok, bad_esc, bad_met)]}")
    assert len(bad_pay) == len(bad_cw) == len(bad_ok) == len(bad_esc) == len(bad_met) == 0, msg
    return got


@pytest.fixture(scope="module")
def P(native):
    import paper_1710_08314_b200 as P

    return P


SMALL = [(16, 6, None), (64, 24, "8"), (128, 32, "11:621:0:0:0"), (256, 100, "16-CCITT")]


@pytest.mark.parametrize("prec", ["f32", "i8"])
@pytest.mark.parametrize("n,k,crc", SMALL)
def test_rough_llrs_all_kinds(P, gpu, oracle_lib, n, k, crc, prec):
    """Adversarial LLRs (zeros, ties, saturation) through every decoder kind."""
    rng = np.random.default_rng(1000 + n + (prec == "i8"))
    code = _code(P, n, k, crc)
    llr = rough_llrs(rng, n, 48, prec)
    pruning = P.PruningConfig(rep_max=8) if prec == "i8" else P.PruningConfig()
    for kind in KINDS:
        if P.DecoderKind[kind].uses_crc and not crc:
            continue
        ls = [1] if kind in ("sc", "ssc") else ([2, 8] if kind in ("pa_sscl", "fa_sscl") else [1, 2, 4, 8, 32])
        for l in ls:
            check_parity(P, gpu, code, kind, l, prec, pruning, llr, "rough")


@pytest.mark.parametrize("prec", ["f32", "i8"])
def test_sc_rung_shortcuts_adversarial(P, gpu, oracle_lib, prec):
    """The SC rung's exact shortcuts (rate-1 hard decision unless an input is
    zero, all-frozen sub-nodes, in-lane subtree recursion) under LLRs full of
    zeros, ties and saturation, on large codes of several rates."""
    rng = np.random.default_rng(4242 + (prec == "i8"))
    for n, k, crc in [(1024, 300, "16-CCITT"), (2048, 1723, "32-GZIP"), (2048, 600, "8")]:
        code = _code(P, n, k, crc)
        llr = rough_llrs(rng, n, 40, prec)
        for kind in ("sc", "ssc", "fa_sscl"):
            check_parity(P, gpu, code, kind, 4, prec, P.PruningConfig(), llr, "sc-rough")
        # sparse zeros in otherwise clean frames exercise the zero fallback
        _, clean = P.channel(code, 3.0, 11, 0, 40, prec, 4.0 if prec == "i8" else 0.0)
        clean = clean.copy()
        clean[rng.random(clean.shape) < 0.01] = 0
        check_parity(P, gpu, code, "ssc", 1, prec, P.PruningConfig(), clean, "sc-zeros")


@pytest.mark.parametrize("prec", ["f32", "i8"])
def test_awgn_mid_codes(P, gpu, oracle_lib, prec):
    rng_seed = 7
    for n, k, crc, snr in [(256, 100, "16-CCITT", 2.0), (1024, 480, "32-GZIP", 2.0)]:
        code = _code(P, n, k, crc)
        _, llr = P.channel(code, snr, rng_seed, 0, 64, prec, 4.0 if prec == "i8" else 0.0)
        pr = P.PruningConfig(rep_max=8) if prec == "i8" else P.PruningConfig()
        for kind, l in [("ssc", 1), ("sscl", 4), ("ca_sscl", 8), ("ca_sscl", 16), ("pa_sscl", 8),
                        ("fa_sscl", 32), ("scl", 4)]:
            check_parity(P, gpu, code, kind, l, prec, pr, llr, "awgn")


def test_cfg0_like_f32(P, gpu, oracle_lib):
    """N=2048, K=1723, CRC-32, GA@4.5 dB, CA-SSCL L=4, float, 4.5 dB."""
    code = _code(P, 2048, 1723, "32-GZIP", ga=4.5)
    _, llr = P.channel(code, 4.5, 42, 0, 128, "f32")
    check_parity(P, gpu, code, "ca_sscl", 4, "f32", P.PruningConfig(), llr, "cfg0")


def test_cfg1_like_i8(P, gpu, oracle_lib):
    """Same code, CA-SSCL L=8, int8 scale 4, REP_8-, 3.5 dB: bit-exact."""
    code = _code(P, 2048, 1723, "32-GZIP", ga=4.5)
    _, llr = P.channel(code, 3.5, 42, 0, 128, "i8", 4.0)
    check_parity(P, gpu, code, "ca_sscl", 8, "i8", P.PruningConfig(rep_max=8), llr, "cfg1")


def test_cfg2_like_fa(P, gpu, oracle_lib):
    """Fully adaptive SCL up to Lmax=32, float, at a low SNR (deep ladder)."""
    code = _code(P, 2048, 1723, "32-GZIP", ga=4.5)
    for snr in (2.5, 3.5):
        _, llr = P.channel(code, snr, 42, 0, 48, "f32")
        got = check_parity(P, gpu, code, "fa_sscl", 32, "f32", P.PruningConfig(), llr, f"cfg2@{snr}")
        assert got["esc"].max() >= 2


GOLD = __import__("os").path.join(__import__("os").path.dirname(__file__), "golden")


def _gold_files():
    import glob
    import os

    return sorted(glob.glob(os.path.join(GOLD, "decode_*.npz")))


@pytest.mark.parametrize("path", _gold_files(), ids=lambda p: p.split("decode_")[-1][:-4])
def test_gpu_matches_reference_golden(P, gpu, path):
    """GPU outputs == the UNMODIFIED reference's outputs stored in the golden
    fixtures (no oracle in between)."""
    z = np.load(path)
    n, k, crc = int(z["n"]), int(z["k"]), str(z["crc"]) or None
    c = [int(x) for x in z["pruning"]]
    pr = P.PruningConfig(bool(c[0]), bool(c[1]), bool(c[2]), bool(c[3]), c[4], c[5])
    code = P.make_code(n, k, z["frozen"], crc)
    x = gpu.from_numpy(np.ascontiguousarray(z["llr"])).cuda()
    for j in range(int(z["runs"])):
        kind, l = str(z[f"r{j}_kind"]), int(z[f"r{j}_l"])
        dec = P.FrameDecoder(code, kind, l, str(z["precision"]), pr)
        o = dec.decode_batch(x, codeword=True)
        gpu.cuda.synchronize()
        pb, cb = (code.payload_size + 7) // 8, (n + 7) // 8
        tag = f"{path} {kind} L={l}"
        assert np.array_equal(o["payload"].cpu().numpy()[:, :pb], z[f"r{j}_payload"]), tag
        assert np.array_equal(o["codeword"].cpu().numpy()[:, :cb], z[f"r{j}_codeword"]), tag
        assert np.array_equal(o["crc_ok"].cpu().numpy(), z[f"r{j}_crc_ok"]), tag
        assert np.array_equal(o["esc"].cpu().numpy(), z[f"r{j}_esc"]), tag
        assert np.array_equal(o["metric"].cpu().numpy(), z[f"r{j}_metric"].astype(np.float32)), tag


def _b(s):
    return np.array([c == "1" for c in s], np.uint8)


def test_gpu_pinned_list_cases(P, gpu):
    """test_list.cpp:78-193 pinned single-node decodes through the GPU."""
    none = P.PruningConfig.none()
    r = P.FrameDecoder(P.make_code(2, 1, _b("10")), "scl", 1, "f32", none).decode([-2.0, 5.0])
    assert r.metric == 2.0 and r.codeword.tolist() == [0, 0]
    r = P.FrameDecoder(P.make_code(2, 1, _b("01")), "scl", 2, "f32", none).decode([3.0, 3.0])
    assert r.metric == 0.0 and r.payload.tolist() == [0]
    r = P.FrameDecoder(P.make_code(8, 4, _b("11110000")), "sscl", 1, "f32").decode(
        [1, -2, 3, -4, 100, 100, 100, 100])
    assert r.metric == 6.0
    r = P.FrameDecoder(P.make_code(4, 1, _b("1110")), "sscl", 2, "f32").decode([1, 1, 1, -5])
    assert r.metric == 3.0 and r.codeword.tolist() == [1, 1, 1, 1] and r.payload.tolist() == [1]
    r = P.FrameDecoder(P.make_code(4, 4, _b("0000")), "sscl", 1, "f32").decode([9, -8, 1, -2])
    assert r.codeword.tolist() == [0, 1, 0, 1] and r.metric == 0.0
    spc = P.FrameDecoder(P.make_code(4, 3, _b("1000")), "sscl", 2, "f32")
    r = spc.decode([1, 5, -6, -7])
    assert r.codeword.tolist() == [0, 0, 1, 1] and r.metric == 0.0
    r = spc.decode([1, 5, -6, 7])
    assert r.codeword.tolist() == [1, 0, 1, 0] and r.metric == 1.0
    r = P.FrameDecoder(P.make_code(2, 2, _b("00")), "scl", 2, "f32", none).decode([0.0, 0.0])
    assert r.metric == 0.0 and r.payload.tolist() == [0, 0] and r.codeword.tolist() == [0, 0]


def test_gpu_ml_on_tiny_code(P, gpu):
    """test_list.cpp:291-319 / acceptance criterion 2: a wide list reaches the
    maximum-likelihood codeword of an (8,4) code."""
    import itertools

    fz = P.construct_frozen(8, 4, 0.5)
    code = P.make_code(8, 4, fz)
    book = []
    u = np.zeros(8, np.uint8)
    for bits in itertools.product([0, 1], repeat=4):
        u[:] = 0
        u[code.info_pos] = bits
        x = u.copy()
        inc = 1
        while inc < 8:  # x = u * F^{(x)3} and back: systematic codeword via two transforms
            for i in range(8):
                if i & inc == 0:
                    x[i] ^= x[i + inc]
            inc <<= 1
        x[fz == 1] = 0
        inc = 1
        while inc < 8:
            for i in range(8):
                if i & inc == 0:
                    x[i] ^= x[i + inc]
            inc <<= 1
        book.append(x.copy())
    rng = np.random.default_rng(303)
    llr = rng.integers(-9, 10, (300, 8)).astype(np.float32)
    for l in (8, 16):
        dec = P.FrameDecoder(code, "scl", l, "f32", P.PruningConfig.none())
        o = dec.decode_batch(gpu.from_numpy(llr).cuda(), codeword=True)
        met = o["metric"].cpu().numpy()
        for f in range(300):
            best = min(float(np.abs(llr[f][(x != (llr[f] < 0))]).sum()) for x in book)
            assert met[f] == best


def test_cfg3_mixed_codes_one_batch(P, gpu, oracle_lib, monkeypatch):
    """Mixed-MCS: 31 codes (N 128..1024, CRC-11/24) in one batch with a
    per-frame code id; every frame equals the oracle of its own code."""
    from paper_1710_08314_b200.workload import MixedWorkload, make_batch

    wl = MixedWorkload()
    codes, cid, info, ks, llr = make_batch(wl, 0, 1024)
    assert len(codes) == 31 and len(set(cid.tolist())) == 31
    # CA at L=8 and SSCL at L=2 run several frames per warp (frames bucketed
    # by code); SSC and FA's first pass run the frame-per-lane SC kernel; the
    # last FA case forces the speculative ladder tail (its commit kernel
    # copies each frame's own code's byte counts)
    for kind, l, spec_max in [("ca_sscl", 8, None), ("sscl", 2, None), ("ssc", 1, None), ("fa_sscl", 8, None),
                              ("fa_sscl", 8, "2000"), ("fa_sscl", 32, "2000")]:
        if spec_max:
            monkeypatch.setenv("PLB_SPEC_MAX", spec_max)
        dec = P.FrameDecoder(codes, kind, l, "f32", P.PruningConfig())
        monkeypatch.delenv("PLB_SPEC_MAX", raising=False)
        o = dec.decode_batch(gpu.from_numpy(llr).cuda(), code_id=gpu.from_numpy(cid).cuda(), codeword=True)
        gpu.cuda.synchronize()
        got = {k: v.cpu().numpy() for k, v in o.items() if v is not None}
        for i, c in enumerate(codes):
            rows = np.flatnonzero(cid == i)
            ref = _oracle(c, kind, l, "f32", P.PruningConfig()).decode(np.ascontiguousarray(llr[rows, :c.n]))
            pb, cb = (c.payload_size + 7) // 8, (c.n + 7) // 8
            tag = (kind, l, c.n)
            assert np.array_equal(got["payload"][rows, :pb], ref.payload), tag
            assert np.array_equal(got["codeword"][rows, :cb], ref.codeword), tag
            assert np.array_equal(got["crc_ok"][rows], ref.crc_ok), tag
            assert np.array_equal(got["esc"][rows], ref.esc), tag
            assert np.array_equal(got["metric"][rows], ref.metric.astype(np.float32)), tag


def test_packed_frames_match_padded(P, gpu):
    """Packed variable-length frames (pl_decode_packed, pl_decode_host_packed
    with several chunks) decode exactly as the padded layout, for the mixed
    31-code batch in float and a mixed int8 batch; malformed offsets fail
    with PL_ERR_ARG (ValueError)."""
    import os

    from paper_1710_08314_b200.workload import MixedWorkload, make_batch

    wl = MixedWorkload()
    codes, cid, info, ks, llr = make_batch(wl, 0, 1500)
    cases = [("f32", llr, codes, cid)]
    # int8: N 16..256, every frame 16-byte aligned as packed
    c8 = [_code(P, n, max(4, n // 2 - 8), "8") for n in (16, 64, 256)]
    cid8 = np.random.default_rng(3).integers(0, 3, 900).astype(np.int32)
    llr8 = np.zeros((900, 256), np.int8)
    for i, c in enumerate(c8):
        rows = np.flatnonzero(cid8 == i)
        _, x = P.channel(c, 2.0, 11, 0, rows.size, "i8", 4.0)
        llr8[rows, :c.n] = x
    cases.append(("i8", llr8, c8, cid8))
    for prec, x, cs, ci in cases:
        kind, l = ("ca_sscl", 8) if prec == "f32" else ("fa_sscl", 8)
        dec = P.FrameDecoder(cs, kind, l, prec, P.PruningConfig())
        ref = dec.decode_batch(gpu.from_numpy(np.ascontiguousarray(x)).cuda(),
                               code_id=gpu.from_numpy(ci).cuda())
        gpu.cuda.synchronize()
        ref = {k: v.cpu().numpy() for k, v in ref.items() if v is not None}
        buf, off = dec.pack_frames([x[f, :cs[ci[f]].n] for f in range(x.shape[0])])
        assert buf.size < x.size
        b2, o2 = dec.pack_batch(x, ci)
        assert np.array_equal(b2, buf) and np.array_equal(o2, off)
        o = dec.decode_packed(gpu.from_numpy(buf).cuda(), gpu.from_numpy(off).cuda(),
                              code_id=gpu.from_numpy(ci).cuda())
        gpu.cuda.synchronize()
        hout = {k: np.zeros_like(v) for k, v in ref.items()}
        dec.set_host_chunk(256)  # several chunks
        dec.decode_host_packed_into(buf, off, hout, ci)
        dec.set_host_chunk(0)
        got = {k: o[k].cpu().numpy() for k in ("payload", "crc_ok", "esc", "metric")}
        for k in ("crc_ok", "esc", "metric"):
            assert np.array_equal(got[k], ref[k]), (prec, k)
            assert np.array_equal(hout[k], ref[k]), (prec, k, "host")
        for i, c in enumerate(cs):  # payload bytes past a code's own size are not written
            rows, pb = np.flatnonzero(ci == i), (c.payload_size + 7) // 8
            assert np.array_equal(got["payload"][rows, :pb], ref["payload"][rows, :pb]), (prec, c.n)
            assert np.array_equal(hout["payload"][rows, :pb], ref["payload"][rows, :pb]), (prec, c.n, "host")
        with pytest.raises(ValueError, match="packed frame"):
            bad = off.copy()
            bad[1] = bad[0] + 1  # overlapping and misaligned
            dec.decode_host_packed_into(buf, bad, hout, ci)


def test_decode_host_matches_device_path(P, gpu):
    """pl_decode_host (pageable and pinned buffers, chunked) == pl_decode."""
    import os

    code = _code(P, 1024, 480, "32-GZIP")
    _, llr = P.channel(code, 2.0, 9, 0, 3000, "i8", 4.0)
    dec = P.FrameDecoder(code, "fa_sscl", 16, "i8", P.PruningConfig(rep_max=8))
    o = dec.decode_batch(gpu.from_numpy(llr).cuda())
    gpu.cuda.synchronize()
    dec.set_host_chunk(700)
    h = dec.decode_host(llr)
    for k in ("payload", "crc_ok", "esc", "metric"):
        assert np.array_equal(h[k], o[k].cpu().numpy()), k


def test_edge_codes(P, gpu, oracle_lib):
    """Rate-1 and rate-1/N codes, the smallest N, and the largest N = 16384
    and 32768 at L = 32 (the per-warp area forces 1-warp blocks)."""
    rng = np.random.default_rng(99)
    cases = [
        (P.make_code(64, 56, np.zeros(64, np.uint8), "8"), ["ssc", "sscl", "fa_sscl"]),  # no frozen bit
        (P.make_code(64, 1, np.r_[np.ones(63, np.uint8), 0]), ["sc", "ssc", "scl", "sscl"]),  # repetition code
        (P.make_code(2, 1, np.array([1, 0], np.uint8)), ["sc", "ssc", "scl", "sscl"]),
        (_code(P, 16384, 8000, "32-GZIP"), ["ssc", "fa_sscl"]),
        (_code(P, 32768, 20000, "32-GZIP"), ["ssc", "fa_sscl"]),
    ]
    for code, kinds in cases:
        for prec in ("f32", "i8"):
            llr = rough_llrs(rng, code.n, (3 if code.n > 16384 else 6) if code.n > 4096 else 24, prec)
            for kind in kinds:
                l = 32 if code.n > 4096 else 8
                check_parity(P, gpu, code, kind, l, prec, P.PruningConfig(), llr, "edge")


def test_cfg4_like_l32(P, gpu, oracle_lib):
    code = _code(P, 2048, 1024, "32-GZIP")
    _, llr = P.channel(code, 1.5, 42, 0, 24, "f32")
    check_parity(P, gpu, code, "ca_sscl", 32, "f32", P.PruningConfig(), llr, "cfg4")


@pytest.mark.parametrize("prec", ["f32", "i8"])
def test_alternate_kernels(P, gpu, oracle_lib, prec, monkeypatch):
    """The opt-in / fallback launch paths stay bit-exact: team mode (a block
    of warps per frame at L = 16/32, PLB_TEAM), the warp-per-frame SC kernel
    (PLB_SC_LANES=0), one frame per warp at small L (PLB_FPW=1), the
    regular layout for small passes (PLB_SOLO=0; by default a pass with at
    most one frame per block, as here, runs in solo mode), and the
    several-frames-per-warp plan of small adaptive rungs (PLB_SMALL_RUNGS=0;
    by default a rung with few frames takes the 1-frame-per-warp launch)."""
    code = _code(P, 1024, 480, "32-GZIP")
    _, llr = P.channel(code, 2.0, 5, 0, 96, prec, 4.0 if prec == "i8" else 0.0)
    pr = P.PruningConfig(rep_max=8) if prec == "i8" else P.PruningConfig()
    for env, cases in [({"PLB_TEAM": "4", "PLB_TEAM_L": "16"}, [("ca_sscl", 16), ("ca_sscl", 32)]),
                       ({"PLB_SC_LANES": "0"}, [("ssc", 1), ("fa_sscl", 8)]),
                       ({"PLB_FPW": "1"}, [("ca_sscl", 4), ("sscl", 2)]),
                       ({"PLB_SOLO": "0"}, [("ca_sscl", 8), ("fa_sscl", 32), ("sscl", 2)]),
                       ({"PLB_SMALL_RUNGS": "0"}, [("fa_sscl", 8), ("pa_sscl", 4)])]:
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        for kind, l in cases:
            check_parity(P, gpu, code, kind, l, prec, pr, llr, f"env={env}")
        for k in env:
            monkeypatch.delenv(k)


@pytest.mark.parametrize("prec", ["f32", "i8"])
def test_fa_speculative_tail(P, gpu, oracle_lib, prec, monkeypatch):
    """FA ladder, speculative tail: with at most PLB_SPEC_MAX frames at the
    third-last rung the last three rungs decode side by side into a staging
    area and a commit kernel keeps the first passing list size
    (decoders.hpp:70-82).  The result is the plain ladder's, on both sides
    of the threshold, with the codeword output, for mixed codes, and equal to
    PLB_SPEC=0."""
    scale = {"f32": 0.0, "i8": 4.0}[prec]  # (int16: tests/test_gpu_int16.py, test_gpu_scale_parity.py)
    code = _code(P, 1024, 480, "32-GZIP")
    _, llr = P.channel(code, 1.5, 9, 0, 160, prec, scale)
    pr = P.PruningConfig()
    outs = []
    for env in ({}, {"PLB_SPEC_MAX": "4"}, {"PLB_SPEC_MAX": "1000"}, {"PLB_SPEC": "0"}):
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        for l in (8, 32):
            got = check_parity(P, gpu, code, "fa_sscl", l, prec, pr, llr, f"spec env={env}")
            assert got["esc"].max() == l  # the ladder reached its last rung
            outs.append((l, got))
        for k in env:
            monkeypatch.delenv(k)
    for l, got in outs[2:]:
        base = outs[0][1] if l == 8 else outs[1][1]
        for key in ("payload", "codeword", "crc_ok", "esc", "metric"):
            assert np.array_equal(got[key], base[key]), key


def test_sc_lane_ops_with_zero_llrs(P, gpu, oracle_lib):
    """The float SC pass decides G ops with a rate-1 child in registers
    (OP_GR1) and chains F ops to their producer; a zero among the g values
    of any lane sends the warp through the plain G op and the expanded
    recursion instead.  Frames with planted zeros / equal magnitudes (g = 0)
    and clean frames, both schedules (PLB_LANE_GR1 / PLB_LANE_CHAIN off)."""
    import os

    code = _code(P, 2048, 1723, "32-GZIP", ga=4.5)
    _, llr = P.channel(code, 4.5, 3, 0, 96, "f32")
    llr = llr.copy()
    rng = np.random.default_rng(1)
    for f in range(0, 96, 3):  # every third frame: a[i] = -+b[i] pairs and zeros
        for _ in range(8):
            h = 1 << rng.integers(5, 11)
            i = int(rng.integers(0, 2048 // (2 * h))) * 2 * h + int(rng.integers(0, h))
            llr[f, i + h] = llr[f, i] * (1 if rng.integers(2) else -1)
        llr[f, rng.integers(0, 2048, 4)] = 0.0
    pr = P.PruningConfig()
    ref = None
    for env in ({}, {"PLB_LANE_GR1": "0"}, {"PLB_LANE_CHAIN": "0"}, {"PLB_LANE_GR1": "0", "PLB_LANE_CHAIN": "0"}):
        old = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        try:
            for kind in ("ssc", "fa_sscl"):
                got = check_parity(P, gpu, code, kind, 4 if kind == "fa_sscl" else 1, "f32", pr, llr, f"env={env}")
                if kind == "ssc":
                    if ref is None:
                        ref = got
                    assert np.array_equal(got["payload"], ref["payload"])
        finally:
            for k, v in old.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v


@pytest.mark.parametrize("prec", ["f32", "i8", "i16"])
def test_interleaved_llr_layout(P, gpu, prec):
    """PL_LLR_INTERLEAVED32 (pl_set_llr_layout): the frame-per-lane SC pass
    reads a channel interleaved in groups of 32 frames; same outputs as the
    frame-major layout, a frame count that is not a multiple of 32, short
    codes (a frame shorter than a 16-byte chunk), and the calls that must
    refuse it."""
    scale = {"f32": 0.0, "i8": 4.0, "i16": 64.0}[prec]
    for n, k, crc, nf in [(2048, 1723, "32-GZIP", 1000), (256, 100, "16-CCITT", 77), (8, 4, None, 40)]:
        code = _code(P, n, k, crc)
        _, llr = P.channel(code, 3.0, 11, 0, nf, prec, scale)
        for kind in ("ssc", "sc"):
            dec = P.FrameDecoder(code, kind, 1, prec, P.PruningConfig())
            ref = dec.decode_batch(gpu.from_numpy(llr).cuda(), codeword=True)
            gpu.cuda.synchronize()
            ref = {k_: v.cpu().numpy().copy() for k_, v in ref.items() if v is not None}
            dec.set_llr_layout(True)
            got = dec.decode_batch(gpu.from_numpy(P.interleave32(llr)).cuda(), codeword=True, nframes=nf)
            gpu.cuda.synchronize()
            for key, r in ref.items():
                assert np.array_equal(got[key].cpu().numpy()[:nf], r), (n, kind, key)
            with pytest.raises(P.ConfigError):
                dec.decode_host(llr)
            dec.set_llr_layout(False)
    code = _code(P, 256, 100, "16-CCITT")
    with pytest.raises(P.ConfigError):
        P.FrameDecoder(code, "ca_sscl", 4, prec, P.PruningConfig()).set_llr_layout(True)


@pytest.mark.parametrize("prec", ["f32", "i8"])
def test_ragged_and_empty_batches(P, gpu, oracle_lib, prec):
    """Batch sizes that leave warps, sub-warps (2 / 4 frames per warp at small
    L) and the 32-frame groups of the frame-per-lane SC pass partly filled —
    1, 3, 31, 33, 65 frames — decode exactly like the oracle through every
    kind; an empty batch is a no-op on the device and the host path."""
    code = _code(P, 256, 100, "16-CCITT")
    rng = np.random.default_rng(5)
    full = rough_llrs(rng, code.n, 65, prec)
    for kind, l in (("ssc", 1), ("ca_sscl", 2), ("ca_sscl", 8), ("pa_sscl", 4), ("fa_sscl", 8)):
        for nf in (1, 3, 31, 33, 65):
            check_parity(P, gpu, code, kind, l, prec, P.PruningConfig(), full[:nf], f"ragged nf={nf}")
        dec = P.FrameDecoder(code, kind, l, prec, P.PruningConfig())
        out = dec.decode_batch(gpu.from_numpy(full[:0].copy()).cuda())
        gpu.cuda.synchronize()
        assert out["payload"].shape[0] == 0 and out["crc_ok"].shape[0] == 0
        hout = dec.decode_host(full[:0].copy())
        assert hout["payload"].shape[0] == 0
        # ... and the handle still decodes afterwards
        check_parity(P, gpu, code, kind, l, prec, P.PruningConfig(), full[:5], "after empty")
