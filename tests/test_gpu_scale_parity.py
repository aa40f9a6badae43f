"""At-scale parity against the compiled, unmodified reference (oracle/_ref):
every BASELINE config at its exact shape, >= 4096 frames per case, all
decoded by the sm_100a path through the C ABI and by the reference's own
FrameDecoder<R> on identical LLR bytes.  Per frame: payload, codeword,
crc_ok, escalation level and the path metric, all bit-exact (the float
metric included; north_star allows 1e-5 relative, the kernels meet 0).
The model is the reference's own equivalence gate, 10 000 frames per code
length (acceptance.cpp:155-226).

Frames are a window of the bench batch of each workload (global frame
indices frame0 .. frame0+4095 of seed 42), so this is the same data the
bench line's `parity_vs_reference` sample covers, at another offset.
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

NFRAMES = 4096
FRAME0 = 100_000
CASES = ["cfg0", "cfg1", "cfg2_2.5", "cfg2_3.5", "cfg2_4.5", "fa_i8_4.5", "fa_i16_4.5",
         "cfg4_L8", "cfg4_L16", "cfg4_L32"]


@pytest.fixture(scope="module")
def P(native):
    import paper_1710_08314_b200 as P

    return P


def _reference(ref_lib, codes, cid, llr, wl):
    nf = llr.shape[0]
    pb = max((c.payload_size + 7) // 8 for c in codes)
    cb = max((c.n + 7) // 8 for c in codes)
    out = {"payload": np.zeros((nf, pb), np.uint8), "codeword": np.zeros((nf, cb), np.uint8),
           "crc_ok": np.zeros(nf, np.uint8), "esc": np.zeros(nf, np.uint8),
           "metric": np.zeros(nf, np.float64)}
    groups = [(0, np.arange(nf))] if cid is None else [(i, np.flatnonzero(cid == i)) for i in range(len(codes))]
    for i, rows in groups:
        if rows.size == 0:
            continue
        c = codes[i]
        ref = ref_lib.Reference(c.n, c.k, c.frozen, c.crc.raw() if c.crc else "", wl.kind, wl.l,
                                wl.precision, wl.pruning.as_tuple())
        r = ref.decode(np.ascontiguousarray(llr[rows, :c.n]), os.cpu_count() or 1)
        out["payload"][rows, :r.payload.shape[1]] = r.payload
        out["codeword"][rows, :r.codeword.shape[1]] = r.codeword
        out["crc_ok"][rows], out["esc"][rows], out["metric"][rows] = r.crc_ok, r.esc, r.metric
    return out


def _compare(got, ref, codes, cid, label):
    nf = ref["esc"].size
    bad = {}
    for key in ("payload", "codeword"):
        # each frame's own bytes (mixed batches: rows are as wide as the widest code)
        bad[key] = np.zeros(nf, bool)
        for i, c in enumerate(codes):
            rows = np.arange(nf) if cid is None else np.flatnonzero(cid == i)
            w = (c.payload_size if key == "payload" else c.n) + 7 >> 3
            bad[key][rows] = (got[key][rows, :w] != ref[key][rows, :w]).any(1)
    bad["crc_ok"] = got["crc_ok"] != ref["crc_ok"]
    bad["esc"] = got["esc"] != ref["esc"]
    bad["metric"] = got["metric"] != ref["metric"].astype(np.float32)
    msg = f"{label}: " + ", ".join(f"{k} {int(v.sum())}/{nf}" for k, v in bad.items())
    assert not any(v.any() for v in bad.values()), msg


@pytest.mark.parametrize("name", CASES)
def test_baseline_config_vs_reference(P, gpu, ref_lib, name):
    from paper_1710_08314_b200.workload import WORKLOADS, make_batch

    wl = WORKLOADS[name]
    codes, cid, info, ks, llr = make_batch(wl, FRAME0, NFRAMES, nthreads=os.cpu_count() or 1)
    dec = P.FrameDecoder(codes, wl.kind, wl.l, wl.precision, wl.pruning)
    out = dec.decode_batch(gpu.from_numpy(llr).cuda(), codeword=True)
    gpu.cuda.synchronize()
    got = {k: v.cpu().numpy() for k, v in out.items() if v is not None}
    ref = _reference(ref_lib, codes, cid, llr, wl)
    _compare(got, ref, codes, cid, name)
    if wl.kind == "fa_sscl":
        # the escalation histogram shows which rungs this case exercised
        hist = np.bincount(got["esc"], minlength=wl.l + 1)
        if name == "cfg2_2.5":
            assert all(hist[l] > 0 for l in (1, 2, 4, 8, 16, 32)), hist


def test_cfg3_mixed_codes_packed_host_path_vs_reference(P, gpu, ref_lib):
    """configs[3] (31 codes, N 128..1024, CRC-11/24, CA-SCL L=8 f32 @ 3 dB)
    through pl_decode_host_packed (host buffers, frames packed at their own
    n) and through pl_decode (padded, device-resident)."""
    from paper_1710_08314_b200.workload import WORKLOADS, make_batch

    wl = WORKLOADS["cfg3"]
    codes, cid, info, ks, llr = make_batch(wl, FRAME0, NFRAMES, nthreads=os.cpu_count() or 1)
    assert np.unique(cid).size == len(codes) == 31
    dec = P.FrameDecoder(codes, wl.kind, wl.l, wl.precision, wl.pruning)
    pk, off = dec.pack_batch(llr, cid)
    o = {"payload": np.zeros((NFRAMES, dec.payload_stride), np.uint8),
         "codeword": np.zeros((NFRAMES, dec.codeword_stride), np.uint8),
         "crc_ok": np.zeros(NFRAMES, np.uint8), "esc": np.zeros(NFRAMES, np.uint8),
         "metric": np.zeros(NFRAMES, np.float32)}
    dec.decode_host_packed_into(pk, off, o, cid)
    ref = _reference(ref_lib, codes, cid, llr, wl)
    _compare(o, ref, codes, cid, "cfg3 packed host")
    out = dec.decode_batch(gpu.from_numpy(llr).cuda(), code_id=gpu.from_numpy(cid).cuda(),
                           codeword=True)
    gpu.cuda.synchronize()
    _compare({k: v.cpu().numpy() for k, v in out.items() if v is not None}, ref, codes, cid,
             "cfg3 padded device")


def test_host_buffer_checks(P, gpu):
    """decode_host* reject LLRs of the wrong dtype / layout and outputs too
    small for the batch instead of reading or writing past them."""
    from paper_1710_08314_b200.workload import WORKLOADS

    wl = WORKLOADS["cfg1"]
    dec = P.FrameDecoder(wl.code(), wl.kind, wl.l, wl.precision, wl.pruning)
    nf = 8
    good = np.zeros((nf, dec.llr_stride), np.int8)
    o = {"payload": np.zeros((nf, dec.payload_stride), np.uint8), "crc_ok": np.zeros(nf, np.uint8),
         "esc": np.zeros(nf, np.uint8), "metric": np.zeros(nf, np.float32)}
    dec.decode_host_into(good, o)
    with pytest.raises(ValueError):
        dec.decode_host_into(good.astype(np.float32), o)
    with pytest.raises(ValueError):
        dec.decode_host_into(np.asfortranarray(good.reshape(nf * 4, -1)), o)
    with pytest.raises(ValueError):
        dec.decode_host_into(good, {**o, "metric": np.zeros(nf - 1, np.float32)})
    with pytest.raises(ValueError):
        dec.decode_host_into(good[:, :-1].copy(), o)
    r = dec.decode_host(good.astype(np.float64))  # converted, not misread
    assert r["esc"].shape == (nf,)
