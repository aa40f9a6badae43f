"""Randomised parity: seeded random codes (N, K, frozen set, CRC preset or
random spec), decoder kinds, list sizes, pruning caps and precisions, with
adversarial or channel LLRs, each decoded on the GPU and by the oracle (the
compiled reference for int16): every output bit-exact."""
import numpy as np
import pytest

from conftest import rough_llrs
from test_gpu_parity import check_parity

pytestmark = pytest.mark.gpu

KINDS = ["sc", "ssc", "scl", "sscl", "ca_sscl", "pa_sscl", "fa_sscl"]
CRCS = [None, "8", "16-CCITT", "32-GZIP", "11:621:0:0:0", "24:b2b117:0:0:0", "5:15:1:1f:0"]


@pytest.fixture(scope="module")
def P(native):
    import paper_1710_08314_b200 as P

    return P


def _random_case(P, rng):
    n = int(2 ** rng.integers(3, 11))
    crc = CRCS[int(rng.integers(len(CRCS)))]
    w = P.CrcSpec.parse(crc).width if crc else 0
    if w >= n - 1:
        crc, w = None, 0
    k = int(rng.integers(1, n - w + 1))
    if rng.random() < 0.5:
        fz = P.construct_frozen(n, k + w, float(rng.uniform(0.05, 0.6)))
    else:  # an arbitrary frozen set
        fz = np.ones(n, np.uint8)
        fz[rng.choice(n, k + w, replace=False)] = 0
    code = P.make_code(n, k, fz, crc)
    kinds = [k_ for k_ in KINDS if crc or not P.DecoderKind[k_].uses_crc]
    kind = kinds[int(rng.integers(len(kinds)))]
    lo = 1 if kind in ("pa_sscl", "fa_sscl") else 0
    l = int(2 ** rng.integers(lo, 6))
    prec = ["f32", "i8", "i16"][int(rng.integers(3))]
    pr = P.PruningConfig(bool(rng.random() < 0.9), bool(rng.random() < 0.9), bool(rng.random() < 0.9),
                         bool(rng.random() < 0.9), int(rng.choice([0, 2, 4, 8, 16])),
                         int(rng.choice([0, 4, 8, 32])))
    return code, kind, l, prec, pr


@pytest.mark.parametrize("seed", range(int(__import__("os").environ.get("PLB_RANDOM_CASES", "200"))))
def test_random_configuration(P, gpu, oracle_lib, ref_lib, seed):
    rng = np.random.default_rng(9000 + seed)
    code, kind, l, prec, pr = _random_case(P, rng)
    nf = 24
    if rng.random() < 0.5:
        llr = rough_llrs(rng, code.n, nf, "i8" if prec == "i8" else "f32")
        if prec == "i16":
            llr = (llr * 256).astype(np.int16)
    else:
        _, llr = P.channel(code, float(rng.uniform(0.0, 4.0)), int(seed), 0, nf, prec,
                           4.0 if prec == "i8" else 0.0)
    label = f"random#{seed} n={code.n} k={code.k} crc={code.crc.raw() if code.crc else None} {pr}"
    if prec != "i16":
        check_parity(P, gpu, code, kind, l, prec, pr, llr, label)
        return
    dec = P.FrameDecoder(code, kind, l, prec, pr)
    o = dec.decode_batch(gpu.from_numpy(np.ascontiguousarray(llr)).cuda(), codeword=True)
    gpu.cuda.synchronize()
    ref = ref_lib.Reference(code.n, code.k, code.frozen, code.crc.raw() if code.crc else "", kind, l,
                            prec, pr.as_tuple()).decode(np.ascontiguousarray(llr), nthreads=8)
    pb, cb = (code.payload_size + 7) // 8, (code.n + 7) // 8
    got = {k: v.cpu().numpy() for k, v in o.items() if v is not None}
    assert np.array_equal(got["payload"][:, :pb], ref.payload), label
    assert np.array_equal(got["codeword"][:, :cb], ref.codeword), label
    assert np.array_equal(got["crc_ok"], ref.crc_ok), label
    assert np.array_equal(got["esc"], ref.esc), label
    assert np.array_equal(got["metric"], ref.metric.astype(np.float32)), label
