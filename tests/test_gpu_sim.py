"""Monte-Carlo points on the GPU against the reference's run_montecarlo
(SURVEY §8(f) #2): with the FrameRng-exact host channel the frame, bit-error,
frame-error and escalation counts are identical, the stop rule included and
for any device chunking; the device (Philox) channel agrees statistically."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S(native):
    from paper_1710_08314_b200 import sim

    return sim


def _code(P, n, k, crc):
    w = P.CrcSpec.parse(crc).width if crc else 0
    return P.make_code(n, k, P.construct_frozen(n, k + w, 0.5), crc)


def _ref(code, cfg, ref_lib):
    crc = code.crc.raw() if code.crc else ""
    return ref_lib.ref_montecarlo(code.n, code.k, code.frozen, crc, cfg.decoder, cfg.list_size,
                                  cfg.precision, cfg.pruning.as_tuple(), cfg.ebn0_min, cfg.ebn0_max,
                                  cfg.ebn0_step, cfg.max_frames, cfg.max_fe, cfg.seed,
                                  cfg.quant_scale, workers=16)


CASES = [
    # (n, k, crc, decoder, L, precision, ebn0 range, max_frames, max_fe)
    (256, 100, "16-CCITT", "ssc", 1, "f32", (1.0, 3.0, 1.0), 20000, 150),
    (128, 48, "8", "fa_sscl", 8, "i8", (1.5, 2.5, 0.5), 6144, 0),
    (512, 256, "32-GZIP", "ca_sscl", 4, "f32", (2.0, 2.0, 1.0), 5000, 40),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[3]}-L{c[4]}-{c[5]}-n{c[0]}")
def test_sim_points_equal_reference(P, S, ref_lib, case):
    n, k, crc, dec, l, prec, (e0, e1, es), mf, mfe = case
    code = _code(P, n, k, crc)
    pr = P.PruningConfig(rep_max=8) if prec == "i8" else P.PruningConfig()
    cfg = S.SimConfig(code, dec, l, prec, pruning=pr, ebn0_min=e0, ebn0_max=e1, ebn0_step=es,
                      max_frames=mf, max_fe=mfe, channel="host", chunk_frames=3072)
    got = S.run_montecarlo(cfg)
    ref = _ref(code, cfg, ref_lib)
    assert len(got) == len(ref)
    for g, r in zip(got, ref):
        assert g.ebn0_db == r[0]
        assert (g.frames, g.bit_errors, g.frame_errors) == (int(r[1]), int(r[2]), int(r[3])), (g, r)
        assert g.esc_mean == r[6]
        if mfe:  # the stop rule fired at the reference's batch boundary
            assert g.frames % 1024 == 0 or g.frames == mf


def test_chunking_does_not_change_counts(P, S):
    code = _code(P, 256, 100, "16-CCITT")
    base = None
    for chunk in (1024, 5000, 0):
        cfg = S.SimConfig(code, "ssc", 1, "f32", ebn0_min=1.5, ebn0_max=1.5, max_frames=30000,
                          max_fe=90, channel="host", chunk_frames=chunk)
        p = S.run_montecarlo(cfg)[0]
        t = (p.frames, p.bit_errors, p.frame_errors)
        assert base is None or t == base, chunk
        base = t


def test_device_channel_statistically_equivalent(P, S):
    code = _code(P, 256, 128, "16-CCITT")
    fer = {}
    for ch in ("host", "device"):
        cfg = S.SimConfig(code, "ca_sscl", 8, "f32", ebn0_min=1.5, ebn0_max=1.5,
                          max_frames=40960, max_fe=0, channel=ch)
        p = S.run_montecarlo(cfg)[0]
        assert p.frames == 40960
        fer[ch] = p.fer
    pbar = (fer["host"] + fer["device"]) / 2
    sd = math.sqrt(2 * pbar * (1 - pbar) / 40960)
    assert abs(fer["host"] - fer["device"]) < 4.5 * sd, fer
    assert 0.005 < pbar < 0.5  # a meaningful operating point


def test_sharded_point_equals_single(P, S):
    """Frame-range shards (multi-GPU) summed == one run (counts are keyed by
    global frame index)."""
    code = _code(P, 256, 100, "16-CCITT")
    cfg = S.SimConfig(code, "sscl", 4, "f32", ebn0_min=2.0, ebn0_max=2.0, max_frames=12288,
                      max_fe=0, channel="device")
    whole = S.run_montecarlo(cfg)[0]
    parts = []
    for r in range(3):
        parts.append(S.run_montecarlo(cfg, rank=r, world=3, reduce=lambda v, op="sum", r=r: v)[0])
    assert sum(p.frames for p in parts) == whole.frames
    assert sum(p.bit_errors for p in parts) == whole.bit_errors
    assert sum(p.frame_errors for p in parts) == whole.frame_errors
    assert sum(p.esc_sum for p in parts) == whole.esc_sum


@pytest.fixture(scope="module")
def P(native):
    import paper_1710_08314_b200 as P

    return P


def test_sweep_cli_two_ranks_equals_one(tmp_path):
    """`python -m paper_1710_08314_b200.sim` under torchrun: each rank takes
    its frame range and the counters are all-reduced; the report equals the
    single-process one (gloo when the ranks share one GPU)."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    args = ["-m", "paper_1710_08314_b200.sim", "256:128:16-CCITT", "--design", "bhat@0.5", "--decoder", "ca_sscl", "--list-size", "4", "--ebn0", "1.0", "2.0", "0.5",
            "--frames", "24576"]
    one = subprocess.run([sys.executable, *args], cwd=root, capture_output=True, text=True,
                         timeout=600)
    assert one.returncode == 0, one.stderr[-2000:]
    two = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes", "1",
                          "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
                          "--master-port", "29571", *args], cwd=root, capture_output=True,
                         text=True, timeout=600)
    assert two.returncode == 0, two.stderr[-2000:]

    def counts(text):
        rows = [r.split(",") for r in text.splitlines() if r and r[0].isdigit()]
        return [(r[0], r[1], r[2], r[3], r[9]) for r in rows]  # all but the timing columns

    assert counts(one.stdout) == counts(two.stdout) and len(counts(one.stdout)) == 3


def test_frame_latency(P, S, gpu):
    """pl_frame_latency: per-frame device decode time (the reference times
    every decode() call, sim.cpp:54-61).  Every frame gets a positive time;
    frames that climbed the FA ladder took longer than SC-only ones; the
    Monte-Carlo point reports the per-frame mean and worst."""
    code = _code(P, 1024, 480, "32-GZIP")
    _, llr = P.channel(code, 2.0, 5, 0, 4096, "f32")
    dec = P.FrameDecoder(code, "fa_sscl", 16, "f32")
    lat = gpu.zeros(4096, dtype=gpu.int32, device="cuda")
    dec.frame_latency(lat)
    out = dec.decode_batch(gpu.from_numpy(llr).cuda())
    gpu.cuda.synchronize()
    t = lat.cpu().numpy().astype(np.int64)
    esc = out["esc"].cpu().numpy()
    assert (t > 0).all()
    assert (esc > 1).any() and (esc == 1).any()
    assert t[esc > 1].mean() > t[esc == 1].mean()
    dec.frame_latency(None)
    lat.zero_()
    dec.decode_batch(gpu.from_numpy(llr).cuda())
    gpu.cuda.synchronize()
    assert int(lat.abs().sum()) == 0
    cfg = S.SimConfig(code, "fa_sscl", 16, "f32", ebn0_min=2.0, ebn0_max=2.0, max_frames=8192,
                      max_fe=0, channel="device")
    p = S.run_montecarlo(cfg)[0]
    assert 0 < p.lat_avg_us <= p.lat_worst_us
