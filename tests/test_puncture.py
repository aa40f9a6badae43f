"""Puncturing / shortening (code.hpp:13-41, channel.hpp:62-89):
the host channel's LLRs with a PuncturePattern are byte-identical to the
reference's transmit (punctured -> 0, shortened -> the largest value, noise
drawn over transmitted positions only, rate = K / transmitted), puncture
files load like load_puncture_file, and punctured frames decode bit-exactly
on the GPU."""
import numpy as np
import pytest


@pytest.fixture(scope="module")
def P(native):
    import paper_1710_08314_b200 as P

    return P


def _pattern(rng, n, npunct, nshort):
    use = np.zeros(n, np.uint8)
    idx = rng.permutation(n)
    use[idx[:npunct]] = 1
    use[idx[npunct:npunct + nshort]] = 2
    return use


def _code(P, n, k, crc, use):
    w = P.CrcSpec.parse(crc).width if crc else 0
    return P.make_code(n, k, P.construct_frozen(n, k + w, 0.5), crc, punct=use)


@pytest.mark.parametrize("prec", ["f32", "i8", "i16"])
def test_punctured_channel_matches_reference(P, ref_lib, prec):
    rng = np.random.default_rng(11)
    for n, k, crc in [(64, 24, "8"), (256, 100, "16-CCITT"), (1024, 500, "32-GZIP")]:
        use = _pattern(rng, n, n // 8, n // 16)
        code = _code(P, n, k, crc, use)
        assert code.rate() == k / int((use == 0).sum())
        info, llr = P.channel(code, 2.0, 7, 50, 24, prec)
        punct = "".join("TPS"[u] for u in use)
        rinfo, rllr = ref_lib.ref_channel(n, k, code.frozen, code.crc.raw(), 2.0, 7, 50, 24, prec,
                                          punct=punct)
        assert np.array_equal(info, rinfo)
        assert np.array_equal(llr, rllr), (n, prec)
        big = {"f32": 1e9, "i8": 127, "i16": 32767}[prec]
        assert np.all(llr[:, use == 1] == 0) and np.all(llr[:, use == 2] == big)


def test_puncture_validation(P):
    fz = P.construct_frozen(16, 10, 0.5)
    with pytest.raises(P.ConfigError):
        P.make_code(16, 10, fz, None, punct="T" * 15)
    with pytest.raises(P.ConfigError):
        P.make_code(16, 10, fz, None, punct="T" * 9 + "P" * 7)  # 9 < K
    P.make_code(16, 10, fz, None, punct="T" * 10 + "PPPSSS")


def test_puncture_files_match_reference(P, ref_lib, tmp_path):
    good = tmp_path / "p.txt"
    good.write_text("8\nTTPTSTTP\n")
    assert np.array_equal(P.load_puncture_file(good), ref_lib.ref_puncture_load(good))
    for i, text in enumerate(["", "x\nTT\n", "8\n", "8\nTTPT\n", "4\nTTXT\n"]):
        path = tmp_path / f"bad{i}.txt"
        path.write_text(text)
        with pytest.raises(RuntimeError) as r:
            ref_lib.ref_puncture_load(path)
        with pytest.raises(P.ParseError) as ours:
            P.load_puncture_file(path)
        assert r.value.args == ("parse", str(ours.value))


@pytest.mark.gpu
def test_punctured_frames_decode_bit_exact(P, gpu, oracle_lib):
    from test_gpu_parity import check_parity

    rng = np.random.default_rng(3)
    for prec in ("f32", "i8"):
        n, k, crc = 256, 100, "16-CCITT"
        code = _code(P, n, k, crc, _pattern(rng, n, 24, 16))
        _, llr = P.channel(code, 1.5, 21, 0, 64, prec)
        pr = P.PruningConfig(rep_max=8) if prec == "i8" else P.PruningConfig()
        for kind, l in [("ssc", 1), ("ca_sscl", 8), ("fa_sscl", 16)]:
            check_parity(P, gpu, code, kind, l, prec, pr, llr, "punct")


@pytest.mark.gpu
def test_device_channel_punctured_positions(P, gpu):
    rng = np.random.default_rng(4)
    n, k = 512, 200
    use = _pattern(rng, n, 40, 20)
    code = _code(P, n, k, "16-CCITT", use)
    for prec, big in (("f32", 1e9), ("i8", 127), ("i16", 32767)):
        info, llr = P.channel_device(code, 2.0, 5, 0, 256, prec)
        x = llr.cpu().numpy()
        assert np.all(x[:, use == 1] == 0) and np.all(x[:, use == 2] == big)
        assert np.all(x[:, use == 0] != 0) if prec == "f32" else True
