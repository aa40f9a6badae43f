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


def test_cfg4_like_l32(P, gpu, oracle_lib):
    code = _code(P, 2048, 1024, "32-GZIP")
    _, llr = P.channel(code, 1.5, 42, 0, 24, "f32")
    check_parity(P, gpu, code, "ca_sscl", 32, "f32", P.PruningConfig(), llr, "cfg4")
