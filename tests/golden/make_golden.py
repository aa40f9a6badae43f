#!/usr/bin/env python
"""Generate the golden vectors in tests/golden/ from the UNMODIFIED reference.

Runs here (where /root/reference exists): builds oracle/_ref from the
reference sources and records, for seeded inputs,
  * CRC check values and CRCs of random messages (CrcEngine::compute),
  * decode trees (PruneTree) for several masks and pruning configs,
  * channel frames (FrameRng / encode_systematic / transmit),
  * full decodes (FrameDecoder<R>::decode) for every decoder kind, both
    precisions, adversarial and AWGN inputs, including the BASELINE codes.
The fixtures are small .npz files; nothing under /root/reference is copied.

  python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402

KINDS = ["sc", "ssc", "scl", "sscl", "ca_sscl", "pa_sscl", "fa_sscl"]
CRC_SPECS = {
    "32-GZIP": (32, 0x04C11DB7, 1, 0xFFFFFFFF, 0xFFFFFFFF),
    "16-CCITT": (16, 0x1021, 0, 0xFFFF, 0),
    "8": (8, 0x07, 0, 0, 0),
    "11:621:0:0:0": (11, 0x621, 0, 0, 0),
    "24:b2b117:0:0:0": (24, 0xB2B117, 0, 0, 0),
    "24:864cfb:0:b704ce:0": (24, 0x864CFB, 0, 0xB704CE, 0),
}


def rough(rng, n, nf, prec):
    pick = rng.integers(0, 8, (nf, n))
    mag = np.where(pick == 0, 0, np.where(pick == 1, 127, rng.integers(0, 8, (nf, n))))
    s = np.where(rng.integers(0, 2, (nf, n)) == 1, -1, 1)
    v = s * mag
    return v.astype(np.int8) if prec == "i8" else (v * 0.5).astype(np.float32)


def ga_mask(n, reliable, design_db, rate):
    import paper_1710_08314_b200 as P  # host helper; the mask is persisted

    return P.construct_frozen_ga(n, reliable, design_db, rate)


def crc_fixture():
    rng = np.random.default_rng(11)
    msg = np.unpackbits(np.frombuffer(b"123456789", np.uint8))
    out = {}
    for i, (txt, spec) in enumerate(CRC_SPECS.items()):
        out[f"check_{i}_spec"] = np.array(spec, np.uint64)
        out[f"check_{i}_value"] = np.uint64(O.ref_crc(txt, msg))
        lens = [0, 1, 7, 8, 9, 63, 64, 65, 215 * 8 + 3, 1723]
        bits = [rng.integers(0, 2, L).astype(np.uint8) for L in lens]
        out[f"rand_{i}_lens"] = np.array(lens)
        out[f"rand_{i}_bits"] = np.concatenate(bits)
        out[f"rand_{i}_crc"] = np.array([O.ref_crc(txt, b) for b in bits], np.uint64)
    np.savez_compressed(os.path.join(HERE, "crc.npz"), **out)


def tree_fixture():
    rng = np.random.default_rng(12)
    out = {}
    cfgs = [(1, 1, 1, 1, 0, 4), (0, 0, 0, 0, 0, 0), (1, 1, 1, 1, 8, 4), (1, 1, 1, 1, 0, 0),
            (1, 0, 1, 0, 2, 0)]
    idx = 0
    for n in (4, 16, 64, 256, 1024, 2048):
        for _ in range(3):
            rel = int(rng.integers(1, n))
            fz = O.ref_construct_frozen(n, rel, float(rng.choice([0.05, 0.3, 0.5])))
            for c in cfgs:
                out[f"t{idx}_frozen"] = fz
                out[f"t{idx}_cfg"] = np.array(c, np.int32)
                out[f"t{idx}_nodes"] = O.ref_tree(fz, c)
                idx += 1
    out["count"] = np.int64(idx)
    np.savez_compressed(os.path.join(HERE, "trees.npz"), **out)


def channel_fixture():
    n, k, crc = 256, 100, "16-CCITT"
    fz = O.ref_construct_frozen(n, k + 16, 0.5)
    info, llr = O.ref_channel(n, k, fz, crc, 2.0, 42, 1000, 8, "f32")
    info8, llr8 = O.ref_channel(n, k, fz, crc, 2.0, 42, 1000, 8, "i8", 4.0)
    np.savez_compressed(os.path.join(HERE, "channel.npz"), frozen=fz, n=n, k=k, crc=crc,
                        ebn0=2.0, seed=42, frame0=1000, info=info, llr=llr, info8=info8,
                        llr8=llr8, scale8=4.0)


def decode_cases():
    """(name, n, k, crc, mask, precision, llr, kinds/l list, pruning)"""
    rng = np.random.default_rng(13)
    cases = []
    # small codes, adversarial LLRs, every kind
    for n, k, crc in [(8, 4, None), (16, 6, None), (64, 24, "8"), (128, 32, "11:621:0:0:0"),
                      (256, 100, "16-CCITT")]:
        w = CRC_SPECS[crc][0] if crc else 0
        fz = O.ref_construct_frozen(n, k + w, 0.5)
        for prec in ("f32", "i8"):
            pr = (1, 1, 1, 1, 8 if prec == "i8" else 0, 4)
            llr = rough(rng, n, 24, prec)
            runs = []
            for kind in KINDS:
                if kind in ("ca_sscl", "pa_sscl", "fa_sscl") and not crc:
                    continue
                ls = [1] if kind in ("sc", "ssc") else ([2, 8] if kind in ("pa_sscl", "fa_sscl")
                                                         else [1, 2, 4, 8, 32])
                runs += [(kind, l) for l in ls]
            cases.append((f"rough_n{n}_{prec}", n, k, crc, fz, prec, llr, runs, pr))
    # AWGN on mid-size codes
    for n, k, crc, snr in [(256, 100, "16-CCITT", 2.0), (1024, 480, "32-GZIP", 2.0)]:
        w = CRC_SPECS[crc][0]
        fz = O.ref_construct_frozen(n, k + w, 0.5)
        for prec, scale in (("f32", 0.0), ("i8", 4.0)):
            _, llr = O.ref_channel(n, k, fz, crc, snr, 42, 0, 32, prec, scale)
            pr = (1, 1, 1, 1, 8 if prec == "i8" else 0, 4)
            runs = [("ssc", 1), ("sscl", 4), ("ca_sscl", 8), ("ca_sscl", 16), ("pa_sscl", 8),
                    ("fa_sscl", 32), ("scl", 4)]
            cases.append((f"awgn_n{n}_{prec}", n, k, crc, fz, prec, llr, runs, pr))
    # BASELINE code: N=2048, K=1723 + CRC-32, GA@4.5 dB
    fz = ga_mask(2048, 1755, 4.5, 1723 / 2048)
    _, llr = O.ref_channel(2048, 1723, fz, "32-GZIP", 4.5, 42, 0, 24, "f32")
    cases.append(("cfg0_like", 2048, 1723, "32-GZIP", fz, "f32", llr, [("ca_sscl", 4)],
                  (1, 1, 1, 1, 0, 4)))
    _, llr = O.ref_channel(2048, 1723, fz, "32-GZIP", 3.5, 42, 0, 24, "i8", 4.0)
    cases.append(("cfg1_like", 2048, 1723, "32-GZIP", fz, "i8", llr, [("ca_sscl", 8)],
                  (1, 1, 1, 1, 8, 4)))
    _, llr = O.ref_channel(2048, 1723, fz, "32-GZIP", 3.0, 42, 0, 12, "f32")
    cases.append(("cfg2_like", 2048, 1723, "32-GZIP", fz, "f32", llr, [("fa_sscl", 32)],
                  (1, 1, 1, 1, 0, 4)))
    fz2 = O.ref_construct_frozen(2048, 1056, 0.5)
    _, llr = O.ref_channel(2048, 1024, fz2, "32-GZIP", 1.5, 42, 0, 8, "f32")
    cases.append(("cfg4_like", 2048, 1024, "32-GZIP", fz2, "f32", llr, [("ca_sscl", 32)],
                  (1, 1, 1, 1, 0, 4)))
    return cases


def decode_fixture():
    for name, n, k, crc, fz, prec, llr, runs, pr in decode_cases():
        out = {"n": n, "k": k, "crc": crc or "", "frozen": fz, "precision": prec, "llr": llr,
               "pruning": np.array(pr, np.int32)}
        for j, (kind, l) in enumerate(runs):
            ref = O.Reference(n, k, fz, crc or "", kind, l, prec, pr)
            r = ref.decode(llr, 8)
            out[f"r{j}_kind"] = kind
            out[f"r{j}_l"] = l
            out[f"r{j}_payload"] = r.payload
            out[f"r{j}_codeword"] = r.codeword
            out[f"r{j}_crc_ok"] = r.crc_ok
            out[f"r{j}_esc"] = r.esc
            out[f"r{j}_metric"] = r.metric
        out["runs"] = len(runs)
        np.savez_compressed(os.path.join(HERE, f"decode_{name}.npz"), **out)


if __name__ == "__main__":
    O.build_ref()
    crc_fixture()
    tree_fixture()
    channel_fixture()
    decode_fixture()
    total = sum(os.path.getsize(os.path.join(HERE, f)) for f in os.listdir(HERE) if f.endswith(".npz"))
    print(f"golden fixtures written: {total / 1e6:.2f} MB")
