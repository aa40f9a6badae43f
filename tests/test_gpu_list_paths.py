"""The final list of every frame (pl_list_paths) against the reference's
ListDecoder<R> introspection (alive_count / is_alive / metric_of,
list_decoder.hpp:91-93) on identical LLRs: the same slots alive (the
logical slot numbering of the slot assignment) and bit-identical
metrics in every alive slot — every path of the list, not only the picked
one."""
import numpy as np
import pytest

from conftest import rough_llrs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P(native):
    import paper_1710_08314_b200 as P

    return P


def _code(P, n, k, crc):
    w = P.CrcSpec.parse(crc).width if crc else 0
    return P.make_code(n, k, P.construct_frozen(n, k + w, 0.5), crc)


@pytest.mark.parametrize("prec", ["f32", "i8"])
@pytest.mark.parametrize("kind", ["sscl", "ca_sscl", "scl"])
def test_final_list_matches_reference(P, gpu, ref_lib, prec, kind):
    rng = np.random.default_rng(77 + (prec == "i8"))
    code = _code(P, 256, 100, "16-CCITT")
    _, awgn = P.channel(code, 1.5, 3, 0, 24, prec, 4.0 if prec == "i8" else 0.0)
    llr = np.concatenate([awgn, rough_llrs(rng, code.n, 16, prec)])
    nf = llr.shape[0]
    pruning = P.PruningConfig(rep_max=8) if prec == "i8" else P.PruningConfig()
    for l in (2, 4, 8, 16, 32):
        dec = P.FrameDecoder(code, kind, l, prec, pruning)
        alive = gpu.zeros(nf, dtype=gpu.int32, device="cuda")
        metric = gpu.full((nf, l), float("nan"), dtype=gpu.float32, device="cuda")
        dec.list_paths(alive, metric)
        dec.decode_batch(gpu.from_numpy(llr).cuda())
        gpu.cuda.synchronize()
        dec.list_paths(None, None)
        a = alive.cpu().numpy().astype(np.uint32)
        m = metric.cpu().numpy()
        c = code.crc
        ref = ref_lib.Reference(code.n, code.k, code.frozen, c.raw() if c else "", kind, l, prec,
                                pruning.as_tuple())
        for f in range(nf):
            _, _, _, _, ra, rm = ref.list_decode(llr[f], l, kind == "ca_sscl")
            want = sum(1 << s for s in range(l) if ra[s])
            assert a[f] == want, (l, f, bin(a[f]), bin(want))
            for s in range(l):
                if ra[s]:
                    assert m[f, s] == np.float32(rm[s]), (l, f, s, m[f, s], rm[s])


def test_psum_layouts_accepted(P, gpu):
    """FrameDecoder's PsumLayout (list_decoder.hpp:22): copy and shared are
    decision-identical in the reference; both are accepted, same outputs."""
    code = _code(P, 256, 100, "16-CCITT")
    _, llr = P.channel(code, 1.5, 5, 0, 32, "f32")
    x = gpu.from_numpy(llr).cuda()
    a = P.FrameDecoder(code, "ca_sscl", 8, "f32", psum_layout="copy").decode_batch(x)
    b = P.FrameDecoder(code, "ca_sscl", 8, "f32", psum_layout="shared").decode_batch(x)
    gpu.cuda.synchronize()
    for k in ("payload", "crc_ok", "esc", "metric"):
        assert gpu.equal(a[k], b[k]), k
    with pytest.raises(P.ConfigError):
        P.FrameDecoder(code, "ca_sscl", 8, "f32", psum_layout="banked")
