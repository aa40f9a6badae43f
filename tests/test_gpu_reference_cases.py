"""The reference's own decoder test cases, restated as batch properties of
the GPU decoder (through the C ABI): each test names the case of
`proj/tests/test_list.cpp` / `test_sc.cpp` it follows.  They need no oracle:
like the reference's cases they compare decoder variants with one another
and with the sent message.  (Bit-exact parity with the oracle / compiled
reference on the same kinds of inputs: test_gpu_parity.py,
test_gpu_scale_parity.py.)
"""
import numpy as np
import pytest

from conftest import rough_llrs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P(native):
    import paper_1710_08314_b200 as P

    return P


def _rough(rng, n, nframes, prec):
    if prec == "i16":
        return (rough_llrs(rng, n, nframes, "i8").astype(np.int16) * 64).clip(-32767, 32767).astype(np.int16)
    return rough_llrs(rng, n, nframes, prec)


def _run(P, torch, code, kind, l, prec, llr, pruning=None):
    dec = P.FrameDecoder(code, kind, l, prec, pruning if pruning is not None else P.PruningConfig())
    out = dec.decode_batch(torch.from_numpy(np.ascontiguousarray(llr)).cuda(), codeword=True)
    torch.cuda.synchronize()
    r = {k: v.cpu().numpy() for k, v in out.items() if v is not None}
    r["payload_bits"] = P.unpack_msb(r["payload"], code.payload_size)
    return r


def _clean(P, code, nframes, seed, amp=4.0):
    """encode_systematic + a noiseless BPSK channel (x -> +-amp): the host
    channel at a very high Eb/N0 gives the codeword's signs."""
    info, llr = P.channel(code, 60.0, seed, 0, nframes, "f32")
    return info, np.where(llr < 0, -amp, amp).astype(np.float32)


@pytest.mark.parametrize("prec", ["f32", "i8", "i16"])
@pytest.mark.parametrize("n", [4, 16, 64, 256])
def test_list_of_one_equals_sc_on_the_full_tree(P, gpu, n, prec):
    """test_list.cpp:196-228: ListDecoder with L = 1 on the unpruned tree is
    ScDecoder, codeword and payload, on adversarial LLRs."""
    rng = np.random.default_rng(101 + n)
    for reliable in (n // 4, n // 2, n - 1):
        code = P.make_code(n, reliable, P.construct_frozen(n, reliable, 0.5))
        llr = _rough(rng, n, 40, prec)
        sc = _run(P, gpu, code, "sc", 1, prec, llr)
        one = _run(P, gpu, code, "scl", 1, prec, llr)
        assert (sc["codeword"] == one["codeword"]).all()
        assert (sc["payload"] == one["payload"]).all()


@pytest.mark.parametrize("prec", ["f32", "i8", "i16"])
@pytest.mark.parametrize("n", [4, 16, 64, 256])
def test_pruned_sc_equals_unpruned_sc(P, gpu, n, prec):
    """test_sc.cpp:39-74: default, wide (no SPC cap) and capped pruning all
    decode like the full tree, bit for bit."""
    rng = np.random.default_rng(100 + n)
    wide = P.PruningConfig(spc_max=0)
    capped = P.PruningConfig(True, True, True, True, 8, 8)
    for reliable in (n // 4, n // 2, 3 * n // 4, n - 1):
        code = P.make_code(n, reliable, P.construct_frozen(n, reliable, 0.5))
        llr = _rough(rng, n, 40, prec)
        ref = _run(P, gpu, code, "sc", 1, prec, llr)
        for cfg in (P.PruningConfig(), wide, capped):
            fast = _run(P, gpu, code, "ssc", 1, prec, llr, cfg)
            assert (ref["codeword"] == fast["codeword"]).all()
            assert (ref["payload"] == fast["payload"]).all()


def test_sc_recovers_the_message_on_a_clean_channel(P, gpu):
    """test_sc.cpp:76-96."""
    for n in (8, 64, 512):
        k = n // 2
        code = P.make_code(n, k, P.construct_frozen(n, k, 0.5))
        info, llr = _clean(P, code, 20, 77 + n)
        r = _run(P, gpu, code, "ssc", 1, "f32", llr)
        assert (r["payload_bits"][:, :k] == info).all()
        assert (P.unpack_msb(r["codeword"], n) == (llr < 0)).all()


def test_single_path_repetition_follows_the_fold_when_saturated(P, gpu):
    """test_list.cpp:230-252: the (4,1) repetition code at int8 extremes —
    both candidate penalties saturate to 127 and the fold alone decides."""
    code = P.make_code(4, 1, np.array([1, 1, 1, 0], np.uint8))
    rng = np.random.default_rng(7)
    llr = np.concatenate([np.array([[-100, -100, 90, 90]], np.int8),
                          (rng.integers(0, 255, (500, 4)) - 127).astype(np.int8)])
    sc = _run(P, gpu, code, "ssc", 1, "i8", llr)
    one = _run(P, gpu, code, "sscl", 1, "i8", llr)
    assert (sc["codeword"] == one["codeword"]).all()


def test_crc_aided_selection_scans_survivors_in_metric_order(P, gpu):
    """test_list.cpp:358-398."""
    code = P.make_code(64, 24, P.construct_frozen(64, 32, 0.5), "8")
    # noiseless frames decode to the sent payload with a clean CRC and metric 0
    info, llr = _clean(P, code, 20, 505)
    r = _run(P, gpu, code, "ca_sscl", 8, "f32", llr)
    assert r["crc_ok"].all() and (r["metric"] == 0).all()
    assert (r["payload_bits"][:, :24] == info).all()
    # noisy frames: a miss falls back to the plain best path; the selection
    # rescues some frames the plain decoder loses
    info, llr = P.channel(code, 1.0, 506, 0, 500, "f32")
    aided = _run(P, gpu, code, "ca_sscl", 8, "f32", llr)
    plain = _run(P, gpu, code, "sscl", 8, "f32", llr)
    miss = aided["crc_ok"] == 0
    assert miss.any() and (aided["payload"][miss] == plain["payload"][miss]).all()
    sent = (aided["payload_bits"][:, :24] == info).all(1)
    differs = (aided["payload"] != plain["payload"]).any(1)
    assert (~miss & sent & differs).sum() > 0
    # a reported success carries a valid CRC: re-decoding its own clean
    # codeword gives the same payload with crc_ok
    okrows = np.flatnonzero(~miss)
    cw = P.unpack_msb(aided["codeword"][okrows], 64)
    again = _run(P, gpu, code, "ca_sscl", 8, "f32", np.where(cw == 1, -4.0, 4.0).astype(np.float32))
    assert again["crc_ok"].all() and (again["payload"] == aided["payload"][okrows]).all()


def test_adaptive_decoding_escalates_only_on_crc_failure(P, gpu):
    """test_list.cpp:400-446 (CRC-32 keeps undetected passes out of the
    comparison)."""
    code = P.make_code(128, 32, P.construct_frozen(128, 64, 0.5), "32-GZIP")
    info, llr = _clean(P, code, 10, 606)
    rp = _run(P, gpu, code, "pa_sscl", 8, "f32", llr)
    rf = _run(P, gpu, code, "fa_sscl", 8, "f32", llr)
    assert rp["crc_ok"].all() and rf["crc_ok"].all()
    assert (rp["esc"] == 1).all() and (rf["esc"] == 1).all()
    assert (rp["payload"] == rf["payload"]).all()

    info, llr = P.channel(code, 0.0, 607, 0, 1000, "f32")
    rp = _run(P, gpu, code, "pa_sscl", 8, "f32", llr)
    rf = _run(P, gpu, code, "fa_sscl", 8, "f32", llr)
    assert np.isin(rp["esc"], (1, 8)).all()
    assert np.isin(rf["esc"], (1, 2, 4, 8)).all()
    assert (rp["esc"][rf["esc"] == 1] == 1).all()
    both_ok = (rp["crc_ok"] == 1) & (rf["crc_ok"] == 1)
    sent_p = (rp["payload_bits"][:, :32] == info).all(1)
    sent_f = (rf["payload_bits"][:, :32] == info).all(1)
    assert (sent_p[both_ok] == sent_f[both_ok]).all()
    both_bad = (rp["crc_ok"] == 0) & (rf["crc_ok"] == 0)
    assert (rp["payload"][both_bad] == rf["payload"][both_bad]).all()
    assert (rf["esc"] > 1).sum() > 0 and both_bad.sum() > 0


def test_adaptive_decoding_composes_the_single_pass_with_aided_passes(P, gpu):
    """test_list.cpp:448-489: PA = SC then CA-SSCL(L); FA = SC, CA-SSCL(2),
    CA-SSCL(4), each frame stopping at its first CRC pass."""
    code = P.make_code(32, 8, P.construct_frozen(32, 16, 0.5), "8")
    info, llr = P.channel(code, 1.5, 707, 0, 400, "f32")
    rp = _run(P, gpu, code, "pa_sscl", 4, "f32", llr)
    rf = _run(P, gpu, code, "fa_sscl", 4, "f32", llr)
    sc = _run(P, gpu, code, "ssc", 1, "f32", llr)
    two = _run(P, gpu, code, "ca_sscl", 2, "f32", llr)
    full = _run(P, gpu, code, "ca_sscl", 4, "f32", llr)
    sc_ok = rf["esc"] == 1
    assert sc_ok.any() and (~sc_ok).any()
    assert (rp["esc"][sc_ok] == 1).all()
    assert (rp["payload"][sc_ok] == sc["payload"][sc_ok]).all()
    assert (rf["payload"][sc_ok] == sc["payload"][sc_ok]).all()
    bad = ~sc_ok
    assert (rp["esc"][bad] == 4).all()
    assert (rp["payload"][bad] == full["payload"][bad]).all()
    assert (rp["crc_ok"][bad] == full["crc_ok"][bad]).all()
    at2 = bad & (two["crc_ok"] == 1)
    at4 = bad & (two["crc_ok"] == 0)
    assert at2.any() and at4.any()
    assert (rf["esc"][at2] == 2).all() and (rf["payload"][at2] == two["payload"][at2]).all()
    assert (rf["esc"][at4] == 4).all() and (rf["payload"][at4] == full["payload"][at4]).all()


def test_undecodable_frames_drive_the_full_escalation_ladder(P, gpu):
    """test_list.cpp:491-507: all-zero LLRs cannot satisfy a CRC with a
    nonzero init, so every rung runs."""
    code = P.make_code(64, 16, P.construct_frozen(64, 32, 0.5), "16-CCITT")
    llr = np.zeros((33, 64), np.float32)
    rp = _run(P, gpu, code, "pa_sscl", 8, "f32", llr)
    rf = _run(P, gpu, code, "fa_sscl", 8, "f32", llr)
    assert not rp["crc_ok"].any() and not rf["crc_ok"].any()
    assert (rp["esc"] == 8).all() and (rf["esc"] == 8).all()
    assert (rp["payload"] == rf["payload"]).all()


def test_fixed_point_metrics_stay_normalized_and_saturation_safe(P, gpu):
    """test_list.cpp:321-356: mostly saturated inputs push the metric range to
    its limit; every alive path's metric stays in [0, max] and the smallest is 0."""
    code = P.make_code(64, 32, P.construct_frozen(64, 32, 0.5))
    rng = np.random.default_rng(404)
    mag = np.where(rng.integers(0, 3, (100, 64)) > 0, 127, rng.integers(0, 8, (100, 64)))
    v = mag * np.where(rng.integers(0, 2, (100, 64)) == 1, -1, 1)
    for prec, dt, top in (("i8", np.int8, 127), ("i16", np.int16, 32767)):
        dec = P.FrameDecoder(code, "sscl", 8, prec, P.PruningConfig())
        alive = gpu.zeros(100, dtype=gpu.int32, device="cuda")
        metric = gpu.zeros((100, 8), dtype=gpu.float32, device="cuda")
        dec.list_paths(alive, metric)
        dec.decode_batch(gpu.from_numpy(v.astype(dt)).cuda())
        gpu.cuda.synchronize()
        a = alive.cpu().numpy().astype(np.uint32)
        m = metric.cpu().numpy()
        on = ((a[:, None] >> np.arange(8)[None, :]) & 1).astype(bool)
        assert on.any(1).all()
        assert (m[on] >= 0).all() and (m[on] <= top).all()
        assert (np.where(on, m, np.inf).min(1) == 0).all()
        dec.list_paths(None, None)


def test_error_rates_fall_as_the_channel_improves(P, native):
    """test_sim.cpp:110-123."""
    from paper_1710_08314_b200 import sim as S
    code = P.make_code(64, 32, P.construct_frozen(64, 32, 0.5))
    cfg = S.SimConfig(code=code, decoder="ssc", ebn0_min=0.0, ebn0_max=2.5, ebn0_step=2.5,
                      max_frames=4000, max_fe=0)
    pts = S.run_montecarlo(cfg)
    assert len(pts) == 2
    assert pts[0].fer > pts[1].fer and pts[0].ber > pts[1].ber
    assert pts[0].bit_errors <= code.k * pts[0].frame_errors
