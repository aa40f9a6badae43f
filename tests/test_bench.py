"""bench.py's driver contract pieces that run without a GPU, plus the
shared-device multi-rank decode on one GPU.

* `--gpus N` relaunches itself with N ranks; rank r takes global frames
  [r*F, (r+1)*F) and one SUM reduces the counters, so the N-rank totals equal
  one process over N*F frames (the multi-GPU analogue of the reference's
  worker-count independence, test_sim.cpp:37-66).
* The reference arm builds its codes from the committed frozen files and its
  inputs with the reference's own channel: it never maps this repo's library.
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(*args, timeout=600):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                       capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-3000:]
    return json.loads(lines[0])


def test_dry_run_two_ranks_match_one_process(native):
    two = _bench("--gpus", "2", "--dry-run", "--frames", "256")
    one = _bench("--dry-run", "--frames", "512")
    assert two["n_gpus"] == 2 and one["n_gpus"] == 1
    assert two["config"]["global_frames"] == 512
    for k in ("frames", "info_ones", "llr_negative", "llr_byte_sum"):
        assert two[k] == one[k], k


def test_dry_run_mixed_codes_two_ranks(native):
    two = _bench("--gpus", "2", "--dry-run", "--frames", "300", "--workload", "cfg3")
    one = _bench("--dry-run", "--frames", "600", "--workload", "cfg3")
    for k in ("frames", "info_ones", "llr_negative", "llr_byte_sum"):
        assert two[k] == one[k], k


def test_reference_arm_uses_only_the_reference(ref_lib):
    d = _bench("--impl", "reference", "--steps", "1", "--ref-sample", "64", "--extra", "cfg0,cfg3",
               "--parity-sample", "64")
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["native_so_loaded"] == ["oracle/_ref/libpolar_ref.so"], d["native_so_loaded"]
    assert [w["workload"] for w in d["workloads"]] == ["cfg0", "cfg3"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0


def test_reference_inputs_equal_product_inputs(ref_lib, native):
    """The reference arm's codes (frozen files) and frames (reference channel)
    are the product arm's, byte for byte."""
    sys.path.insert(0, ROOT)
    import bench
    from paper_1710_08314_b200.workload import WORKLOADS, make_batch

    for name in ("cfg1", "cfg3"):
        wl = WORKLOADS[name]
        codes_r, cid_r, ks_r, llr_r = bench.reference_inputs(ref_lib, wl, 1000, 96, 4)
        codes, cid, info, ks, llr = make_batch(wl, 1000, 96, nthreads=4)
        assert len(codes) == len(codes_r)
        for c, (n, k, crc, fz) in zip(codes, codes_r):
            assert (c.n, c.k) == (n, k)
            assert np.array_equal(c.frozen, fz)
        if cid is not None:
            assert np.array_equal(cid, cid_r)
        assert np.array_equal(ks, ks_r)
        assert llr.tobytes() == llr_r.tobytes()


def test_frozen_files_are_the_ga_construction(native):
    import paper_1710_08314_b200 as P
    from paper_1710_08314_b200.workload import WORKLOADS, crc_width

    seen = 0
    for wl in WORKLOADS.values():
        for n, k, crc, path in wl.code_specs():
            n2, k2, fz = P.load_frozen_file(path)
            assert (n2, k2) == (n, k + crc_width(crc)), path
            assert np.array_equal(fz, P.construct_frozen_ga(n, k + crc_width(crc), wl.design_db, k / n))
            seen += 1
    assert seen >= 33


@pytest.mark.gpu
def test_two_ranks_on_one_gpu_count_like_one_process(gpu):
    """bench.py --gpus 2 (ranks sharing the box's GPU over gloo): the reduced
    counters equal one process decoding the union of the two frame ranges."""
    args = ["--workload", "cfg0", "--steps", "1", "--warmup", "3", "--e2e-steps", "1",
            "--no-cpu", "--extra", "none"]
    two = _bench("--gpus", "2", "--allow-shared", "--frames", "2048", *args)
    one = _bench("--frames", "4096", *args)
    assert two["n_gpus"] == 2 and two["config"]["global_frames"] == 4096
    for k in ("frames_counted", "frame_errors", "bit_errors", "esc_mean"):
        assert two[k] == one[k], k
    assert "note" in two


@pytest.mark.gpu
def test_nccl_group_on_one_rank(gpu):
    """The N > 1 branch's own collectives on hardware: a 1-rank torchrun with
    PLB_BENCH_FORCE_GROUP=1 initialises the NCCL group (device_id = the rank's
    GPU) and runs the barriers, the MAX of the device-timed step and the SUM of
    the counters through it; the line equals a plain run's counters."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    args = ["--workload", "cfg0", "--frames", "4096", "--steps", "1", "--warmup", "3",
            "--e2e-steps", "1", "--no-cpu", "--extra", "none"]
    env = dict(os.environ, PLB_BENCH_FORCE_GROUP="1", OMP_NUM_THREADS="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node=1", "--master-addr=127.0.0.1", f"--master-port={port}",
                        os.path.join(ROOT, "bench.py"), "--gpus", "1", *args],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-3000:]
    grp = json.loads(lines[0])
    one = _bench(*args)
    assert grp["n_gpus"] == 1 and grp["collectives"] == "nccl"
    assert "cpu_affinity" in grp  # the GPU-local CPU binding of multi-rank runs ran (None: nothing to narrow)
    for k in ("frames_counted", "frame_errors", "bit_errors", "esc_mean"):
        assert grp[k] == one[k], k


def test_multi_rank_batch_fits_host_memory(monkeypatch):
    """fit_frames: one rank keeps its batch; N ranks shrink theirs (to a
    multiple of 4096, never below it) when N stagings would not fit the
    available host memory, and all ranks adopt the smallest proposal."""
    sys.path.insert(0, ROOT)
    import bench
    import psutil
    from paper_1710_08314_b200.workload import WORKLOADS

    class R:
        def __init__(self, ws):
            self.ws = ws

        def max(self, x):  # the other rank proposes 8192 frames
            return max(x, -8192.0) if self.ws == 3 else x

    wl = WORKLOADS["cfg2_4.5"]
    assert bench.fit_frames(wl, wl.frames, R(1)) == wl.frames

    class VM:
        available = 64 << 30

    monkeypatch.setattr(psutil, "virtual_memory", lambda: VM)
    f8 = bench.fit_frames(wl, wl.frames, R(8))
    assert 4096 <= f8 < wl.frames and f8 % 4096 == 0
    assert f8 * wl.n * 4 * 2.5 * 8 <= 0.6 * VM.available
    assert bench.fit_frames(wl, wl.frames, R(3)) == 8192
    VM.available = 4 << 40
    assert bench.fit_frames(wl, wl.frames, R(8)) == wl.frames


def test_extra_workload_defaults():
    """The default run covers every other workload at N=1 and the FA points +
    cfg0 at N>1; 'none' and explicit lists are honoured; the main workload
    is never repeated."""
    sys.path.insert(0, ROOT)
    import argparse

    import bench
    from paper_1710_08314_b200.workload import WORKLOADS

    a = argparse.Namespace(extra=None, workload="cfg1")
    one = bench.extra_list(a, 1)
    assert set(one) == set(WORKLOADS) - {"cfg1"}
    assert bench.extra_list(a, 8) == ["cfg0", "cfg2_4.5", "cfg2_3.5"]
    assert bench.extra_list(argparse.Namespace(extra="none", workload="cfg1"), 1) == []
    assert bench.extra_list(argparse.Namespace(extra="cfg1,cfg3", workload="cfg1"), 1) == ["cfg3"]


def test_crc_width_without_library():
    from paper_1710_08314_b200.workload import crc_width

    assert crc_width("32-GZIP") == 32 and crc_width("11:621:0:0:0") == 11
    assert crc_width("24:b2b117:0:0:0") == 24 and crc_width("") == 0 and crc_width("8") == 8
