"""int16 LLRs (llr.hpp:22-26: saturation at +-32767, default
quantisation scale 64) against the compiled, unmodified reference decoder
(oracle/_ref; the C restatement covers float and int8 only): bit-exact
payload, codeword, CRC flag, escalation level and path metric."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

KINDS = ["sc", "ssc", "scl", "sscl", "ca_sscl", "pa_sscl", "fa_sscl"]


@pytest.fixture(scope="module")
def P(native):
    import paper_1710_08314_b200 as P

    return P


def _code(P, n, k, crc):
    w = P.CrcSpec.parse(crc).width if crc else 0
    return P.make_code(n, k, P.construct_frozen(n, k + w, 0.5), crc)


def _rough_i16(rng, n, nframes):
    """zeros, +-32767 and tiny magnitudes: ties and saturation everywhere"""
    pick = rng.integers(0, 8, (nframes, n))
    mag = np.where(pick == 0, 0, np.where(pick == 1, 32767, rng.integers(0, 8, (nframes, n))))
    mag = np.where(pick == 2, rng.integers(16000, 32768, (nframes, n)), mag)
    s = np.where(rng.integers(0, 2, (nframes, n)) == 1, -1, 1)
    return (s * mag).astype(np.int16)


def _check(P, gpu, ref_lib, code, kind, l, pruning, llr, tag):
    dec = P.FrameDecoder(code, kind, l, "i16", pruning)
    o = dec.decode_batch(gpu.from_numpy(np.ascontiguousarray(llr)).cuda(), codeword=True)
    gpu.cuda.synchronize()
    got = {k: v.cpu().numpy() for k, v in o.items() if v is not None}
    crc = code.crc.raw() if code.crc else ""
    ref = ref_lib.Reference(code.n, code.k, code.frozen, crc, kind, l, "i16",
                            pruning.as_tuple()).decode(np.ascontiguousarray(llr), nthreads=8)
    pb, cb = (code.payload_size + 7) // 8, (code.n + 7) // 8
    t = (tag, kind, l, code.n)
    assert np.array_equal(got["payload"][:, :pb], ref.payload), t
    assert np.array_equal(got["codeword"][:, :cb], ref.codeword), t
    assert np.array_equal(got["crc_ok"], ref.crc_ok), t
    assert np.array_equal(got["esc"], ref.esc), t
    assert np.array_equal(got["metric"], ref.metric.astype(np.float32)), t


@pytest.mark.parametrize("n,k,crc", [(64, 24, "8"), (256, 100, "16-CCITT"), (1024, 480, "32-GZIP")])
def test_int16_rough_all_kinds(P, gpu, ref_lib, n, k, crc):
    rng = np.random.default_rng(77 + n)
    code = _code(P, n, k, crc)
    llr = _rough_i16(rng, n, 40)
    for kind in KINDS:
        for l in ([1] if kind in ("sc", "ssc") else [2, 8, 32]):
            _check(P, gpu, ref_lib, code, kind, l, P.PruningConfig(), llr, "rough")


def test_int16_awgn_channel(P, gpu, ref_lib):
    code = _code(P, 2048, 1723, "32-GZIP")
    for snr in (3.0, 4.0):
        info, llr = P.channel(code, snr, 42, 0, 64, "i16")  # scale 64 (channel.hpp:94-100)
        assert llr.dtype == np.int16 and np.abs(llr).max() <= 32767
        for kind, l in [("ssc", 1), ("ca_sscl", 8), ("fa_sscl", 32)]:
            _check(P, gpu, ref_lib, code, kind, l, P.PruningConfig(), llr, f"awgn{snr}")


def test_int16_host_channel_equals_reference(P, ref_lib):
    """The host channel's int16 LLRs are byte-identical to the reference's
    transmit<int16_t> (quantize, llr.hpp:90-102)."""
    code = _code(P, 256, 100, "16-CCITT")
    info, llr = P.channel(code, 2.0, 9, 100, 32, "i16")
    rinfo, rllr = ref_lib.ref_channel(code.n, code.k, code.frozen, code.crc.raw(), 2.0, 9, 100, 32,
                                      "i16")
    assert np.array_equal(info, rinfo) and np.array_equal(llr, rllr)
