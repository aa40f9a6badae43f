#!/usr/bin/env python
"""Benchmark: decoded information throughput (Gb/s) of the B200 polar decoder.

Default workload = BASELINE.json configs[1]: N=2048, K=1723 (+CRC-32 GZIP),
GA frozen set @4.5 dB, CA-SCL L=8 with R0/R1/REP_8-/SPC4 pruning, int8 LLRs
(x4, saturated to +-127) from BPSK-AWGN at 3.5 dB, 262 144 frames per GPU.
One step = one decode of that batch (inputs resident in HBM for `value`;
host buffers with the copies inside the timed region for `e2e`).
`--workload` selects the other BASELINE configs (cfg0, cfg2_{2.5,3.5,4.5},
cfg3 mixed-MCS, cfg4_L{8,16,32}); `--extra` appends a `workloads` block with
the same measurements of further configs (default: every other workload at
N = 1; cfg0 and the paper's FA-SCL points cfg2 @ 4.5 / 3.5 dB at N > 1).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg1]
  python bench.py --impl reference ...   # the reference's own CPU decoder

Multi-GPU: `--gpus N` without a torchrun environment relaunches itself
under torch.distributed.run with N local ranks, one GPU each (NCCL); rank r
decodes global frames [r*F, (r+1)*F) (weak scaling, shard.frame_range) and
the only collectives are one 4 x i64 counter SUM per workload and the
max-over-ranks of the timed region (sim.cpp:84-109, test_sim.cpp:37-66).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decoded info throughput (Gb/s) N=2048 K=1723"
DATA = "synthetic: BPSK-AWGN frames keyed by (seed 42, global frame index), FrameRng semantics"
# further workloads of the default run: every other BASELINE config at N = 1;
# at N > 1 (the driver's scaling run) the paper's FA points and cfg0, whose
# inputs every rank generates on its share of the host cores
EXTRA_DEFAULT = "cfg0,cfg2_4.5,cfg2_3.5,cfg2_2.5,cfg3,cfg4_L8,cfg4_L16,cfg4_L32,fa_i8_4.5,fa_i16_4.5"
EXTRA_DEFAULT_MULTI = "cfg0,cfg2_4.5,cfg2_3.5"
# ncu counters of the current kernels (profiles/traffic.py); the newest round's file wins
COUNTERS_FILES = [os.path.join(ROOT, "profiles", f) for f in ("r02_traffic.json", "r01_traffic.json")]


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="cfg1")
    ap.add_argument("--extra", default=None,
                    help="comma-separated further workloads for the `workloads` block, or 'none' "
                         f"(default: {EXTRA_DEFAULT} at N=1, {EXTRA_DEFAULT_MULTI} at N>1)")
    ap.add_argument("--extra-steps", type=int, default=5)
    ap.add_argument("--frames", type=int, default=0, help="override frames per GPU")
    ap.add_argument("--e2e-steps", type=int, default=0)
    ap.add_argument("--cpu-sample", type=int, default=16384)
    ap.add_argument("--ref-sample", type=int, default=16384)
    ap.add_argument("--parity-sample", type=int, default=4096)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--allow-shared", action="store_true",
                    help="let more ranks than GPUs share devices over gloo (a path exercise, "
                         "not a scaling number)")
    ap.add_argument("--dry-run", action="store_true",
                    help="the multi-rank plumbing only (launch, frame ranges, input generation, "
                         "counter reduction) with no decode; runs without a GPU")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def relaunch(args) -> int:
    """`--gpus N` outside torchrun: re-exec under torch.distributed.run with
    N local ranks on 127.0.0.1 (rank 0 prints the JSON line)."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__), *sys.argv[1:]]
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "1")
    return subprocess.call(cmd, env=env)


def sample_clocks_start(gpu_index: int):
    f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
    q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    try:
        p = subprocess.Popen(["nvidia-smi", "-i", str(gpu_index), f"--query-gpu={q}",
                              "--format=csv,noheader,nounits", "-lms", "100"],
                             stdout=f, stderr=subprocess.DEVNULL)
    except OSError:
        return None, f
    return p, f


def sample_clocks_stop(p, f):
    if p is None:
        return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
    p.terminate()
    try:
        p.wait(5)
    except subprocess.TimeoutExpired:
        p.kill()
    f.flush()
    f.seek(0)
    rows = [r.split(",") for r in f.read().strip().splitlines() if r.strip()]
    os.unlink(f.name)
    sm, smax, reasons = [], None, set()
    names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    for r in rows:
        r = [x.strip() for x in r]
        if len(r) < 9:
            continue
        try:
            sm.append(float(r[1]))
            smax = float(r[2])
        except ValueError:
            continue
        for nm, v in zip(names, r[5:9]):
            if v.lower().startswith("active"):
                reasons.add(nm)
    return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax,
            "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


def dtype_of(wl):
    return {"i8": "int8", "i16": "int16"}.get(wl.precision, "f32")


def esize(wl):
    return {"f32": 4, "i16": 2}.get(wl.precision, 1)


def ncu_counters(wl):
    """ncu counters of this workload's pass kernels (profiles/traffic.py,
    one committed ncu capture per workload of its default batch): {key:
    counters}, the capture's frame count; None if absent."""
    for path in COUNTERS_FILES:
        try:
            with open(path) as fh:
                t = json.load(fh)[wl.name]
            t["source"] = f"{os.path.relpath(path, ROOT)}: {t['source']}"
            return t
        except (OSError, KeyError, ValueError):
            continue
    return None


def common_config(wl, frames_per_gpu, ws):
    """The config both arms report (the driver compares like with like)."""
    return {**wl.describe(), "frames_per_gpu": frames_per_gpu,
            "global_frames": frames_per_gpu * ws, "parallelism": f"frame-range shards x{ws}",
            "l2": "inputs larger than L2 (%.0f MB per GPU per step)" % (frames_per_gpu * wl.n * esize(wl) / 1e6)}


def mapped_native_libs():
    """The in-tree / oracle .so files this process has mapped."""
    out = set()
    try:
        with open("/proc/self/maps") as fh:
            for line in fh:
                p = line.split()[-1] if line.split() else ""
                if p.endswith(".so") and (p.startswith(ROOT) or "/_ref/" in p):
                    out.add(os.path.relpath(p, ROOT))
    except OSError:
        pass
    return sorted(out)


# --------------------------------------------------------------------------
# the reference's own CPU decoder (checker / baseline; oracle/_ref only)

def reference_decode(O, codes, cid, llr, wl, nthr):
    """The compiled reference FrameDecoder<R> over a batch (per code for
    mixed batches); `codes` = [(n, k, crc text, frozen mask)]. Returns
    payload/crc_ok/esc/metric arrays and the seconds spent decoding."""
    nf = llr.shape[0]
    from paper_1710_08314_b200.workload import crc_width

    pb = max((k + crc_width(c) + 7) // 8 for _, k, c, _ in codes)
    out = {"payload": np.zeros((nf, pb), np.uint8), "crc_ok": np.zeros(nf, np.uint8),
           "esc": np.zeros(nf, np.uint8), "metric": np.zeros(nf, np.float64)}
    secs = 0.0
    groups = [(0, np.arange(nf))] if cid is None else [(i, np.flatnonzero(cid == i)) for i in range(len(codes))]
    for i, rows in groups:
        if rows.size == 0:
            continue
        n, k, crc, fz = codes[i]
        ref = O.Reference(n, k, fz, crc, wl.kind, wl.l, wl.precision, wl.pruning.as_tuple())
        x = np.ascontiguousarray(llr[rows, :n])
        t0 = time.perf_counter()
        r = ref.decode(x, nthr)
        secs += time.perf_counter() - t0
        out["payload"][rows, : r.payload.shape[1]] = r.payload
        out["crc_ok"][rows], out["esc"][rows], out["metric"][rows] = r.crc_ok, r.esc, r.metric
    return out, secs


def reference_inputs(O, wl, frame0, nframes, nthr):
    """Codes and inputs built by the reference alone: frozen masks from the
    committed frozen files (load_frozen_file, code.cpp:164-185) and frames
    from FrameRng / random_payload / encode_systematic / transmit
    (channel.hpp:17-89) -- byte-identical to the product arm's host channel
    (tests/test_oracle.py)."""
    from paper_1710_08314_b200.workload import MixedWorkload

    codes = []
    for n, k, crc, path in wl.code_specs():
        n2, _, fz = O.ref_frozen_load(path)
        assert n2 == n, path
        codes.append((n, k, crc, fz))
    if isinstance(wl, MixedWorkload):
        cid = wl.code_ids(frame0, nframes, len(codes))
        nmax = max(c[0] for c in codes)
        dt = {"f32": np.float32, "i8": np.int8, "i16": np.int16}[wl.precision]
        llr = np.zeros((nframes, nmax), dt)
        ks = np.zeros(nframes, np.int64)
        for i, (n, k, crc, fz) in enumerate(codes):
            rows = np.flatnonzero(cid == i)
            if rows.size:
                _, x = O.ref_channel_ids(n, k, fz, crc, wl.ebn0_db, 42,
                                         rows.astype(np.uint64) + np.uint64(frame0),
                                         wl.precision, wl.scale, nthr)
                llr[rows, :n] = x
                ks[rows] = k
        return codes, cid, ks, llr
    n, k, crc, fz = codes[0]
    _, llr = O.ref_channel(n, k, fz, crc, wl.ebn0_db, 42, frame0, nframes, wl.precision,
                           wl.scale, nthr)
    return codes, None, np.full(nframes, k, np.int64), llr


def run_reference(args):
    """The reference's own CPU decoder (oracle/_ref: FrameDecoder<R> compiled
    from /root/reference/proj), all host threads, bounded sample per step.
    Nothing of this repo's product library is loaded in this process."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    from paper_1710_08314_b200.workload import WORKLOADS
    try:
        from oracle import oracle as O
        O.Reference.lib()
    except Exception as e:  # noqa: BLE001
        print(json.dumps({"impl": "reference", "unavailable": f"oracle/_ref not loadable: {e}"}))
        return 0
    nthr = os.cpu_count() or 1

    def one(wl, nf, steps):
        codes, cid, ks, llr = reference_inputs(O, wl, 0, nf, nthr)
        w = max(nthr, nf // 8)
        reference_decode(O, codes, cid[:w] if cid is not None else None, llr[:w], wl, nthr)  # warm-up
        secs = 0.0
        for _ in range(steps):
            secs += reference_decode(O, codes, cid, llr, wl, nthr)[1]
        dt = secs / steps
        return float(ks.sum()) / dt / 1e9, dt

    wl = WORKLOADS[args.workload]
    nf = args.ref_sample
    gbps, dt = one(wl, nf, args.steps)
    out = {
        "impl": "reference", "metric": METRIC, "value": gbps, "unit": "Gb/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": dtype_of(wl),
        "data": DATA, "config": common_config(wl, args.frames or wl.frames, ws),
        "reference_sample_frames_per_step": nf,
        "cpu_baseline": {"value": gbps, "unit": "Gb/s", "cores": nthr, "kind": "reference",
                         "sample": f"{nf} frames of {wl.name} per step, FrameDecoder<R> per thread"},
        "e2e": {"value": gbps, "unit": "Gb/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    extras = extra_list(args, ws)
    if extras:
        out["workloads"] = []
        for name in extras:
            w2 = WORKLOADS[name]
            g2, dt2 = one(w2, args.parity_sample, 2)
            out["workloads"].append({"workload": name, "config": w2.describe(), "value": g2,
                                     "unit": "Gb/s", "ms_per_step": dt2 * 1e3,
                                     "sample_frames_per_step": args.parity_sample, "cores": nthr})
    out["native_so_loaded"] = mapped_native_libs()
    print(json.dumps(out))
    return 0


# --------------------------------------------------------------------------
# the multi-rank plumbing without a decode (CPU test of the N>1 path)

def run_dry(args):
    ws, rank, _ = dist_env()
    import torch.distributed as dist
    from paper_1710_08314_b200.shard import frame_range
    from paper_1710_08314_b200.workload import WORKLOADS, make_batch

    if ws > 1:
        dist.init_process_group("gloo")
    import torch
    wl = WORKLOADS[args.workload]
    F = args.frames or wl.frames
    frame0, frame1 = frame_range(rank, ws, F)
    _, _, info, ks, llr = make_batch(wl, frame0, F, nthreads=1)
    v = np.array([F, int(info.sum()), int((llr < 0).sum()),
                  int(llr.view(np.uint8).astype(np.int64).sum())], np.int64)
    if ws > 1:
        t = torch.from_numpy(v)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        v = t.numpy()
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": ws, "config": common_config(wl, F, ws),
                          "frames": int(v[0]), "info_ones": int(v[1]), "llr_negative": int(v[2]),
                          "llr_byte_sum": int(v[3])}))
    if ws > 1:
        dist.destroy_process_group()
    return 0


# --------------------------------------------------------------------------
# the B200 arm

def bind_near_gpu(cuda_index: int):
    """Multi-rank runs: keep this rank (its input-generation threads and the
    pinned staging they first-touch) on the CPUs NVML reports as closest to
    its GPU, so the host<->device copies of the e2e leg do not cross sockets.
    Returns a description for the JSON line, or None when nothing was done."""
    try:
        import pynvml
        import torch
        pynvml.nvmlInit()
        try:
            uuid = str(torch.cuda.get_device_properties(cuda_index).uuid)
            h = pynvml.nvmlDeviceGetHandleByUUID(("GPU-" + uuid).encode())
        except Exception:  # noqa: BLE001
            h = pynvml.nvmlDeviceGetHandleByIndex(cuda_index)
        ncpu = os.cpu_count() or 1
        words = pynvml.nvmlDeviceGetCpuAffinity(h, (ncpu + 63) // 64)
        near = {64 * i + b for i, w in enumerate(words) for b in range(64) if (int(w) >> b) & 1}
        cur = os.sched_getaffinity(0)
        want = near & cur
        if len(want) < 2 or want == cur:
            return None
        os.sched_setaffinity(0, want)
        return f"{len(want)} of {len(cur)} cpus (NVML affinity of cuda:{cuda_index})"
    except Exception:  # noqa: BLE001
        return None


class Ranks:
    """Process group plumbing: barrier and max-over-ranks (device-timed)."""

    def __init__(self, args):
        import torch
        import torch.distributed as dist

        self.dist = dist
        self.ws, self.rank, local = dist_env()
        ndev = torch.cuda.device_count()
        if ndev == 0:
            raise SystemExit("bench.py: no CUDA device (the decoder has no CPU path)")
        self.shared = self.ws > ndev
        if self.shared and not args.allow_shared:
            raise SystemExit(f"bench.py: {self.ws} ranks but only {ndev} GPU(s); one rank per GPU "
                             "(pass --allow-shared to exercise the path on shared devices)")
        # PLB_BENCH_FORCE_GROUP=1 under a 1-rank torchrun: the NCCL group, barrier
        # and reductions of the N > 1 path on one GPU (tests/test_gpu_scale_parity.py)
        self.group = self.ws > 1 or (os.environ.get("PLB_BENCH_FORCE_GROUP") == "1"
                                     and "MASTER_ADDR" in os.environ)
        if self.group:
            if self.shared:
                dist.init_process_group("gloo")
            else:
                dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        self.local = local % ndev
        torch.cuda.set_device(self.local)
        self.affinity = bind_near_gpu(self.local) if self.group and not self.shared else None
        self.red_dev = "cpu" if self.shared else f"cuda:{self.local}"

    def barrier(self):
        if self.group:
            self.dist.barrier()

    def max(self, x):
        if not self.group:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64, device=self.red_dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())


def measure(wl, F, steps, warmup, e2e_steps, R: Ranks, peaks, peak_src, min_timed_s=0.0):
    """One workload: device-resident throughput with live per-kernel CUDA-event
    timing, error counters reduced over ranks, e2e through the host API, and
    per-kernel roofline fractions.  Returns (line fields, host state kept for
    the parity / CPU-baseline leg)."""
    import torch

    import paper_1710_08314_b200 as P
    from paper_1710_08314_b200.shard import Counters, all_reduce_counters, frame_range
    from paper_1710_08314_b200.workload import make_batch, schedule_work

    ws, rank, local = R.ws, R.rank, R.local
    frame0, _ = frame_range(rank, ws, F)  # weak scaling: each rank its own global frame range
    codes, cid, info, ks, llr_np = make_batch(wl, frame0, F,
                                              nthreads=max(1, (os.cpu_count() or 1) // ws))
    llr_h = torch.from_numpy(llr_np).pin_memory()
    llr_np = llr_h.numpy()  # one host copy (the pinned one): N ranks x 8.6 GB for cfg2
    llr_d = llr_h.cuda(local)
    cid_h = torch.from_numpy(cid).pin_memory() if cid is not None else None
    cid_d = cid_h.cuda(local) if cid is not None else None
    dec = P.FrameDecoder(codes, wl.kind, wl.l, wl.precision, wl.pruning, device=local)
    out = dec.alloc_outputs(F)
    stream = torch.cuda.current_stream(local)
    bits_per_step = float(ks.sum())

    t_w = time.perf_counter()
    for _ in range(warmup):
        dec.decode_batch(llr_d, code_id=cid_d, out=out)
    torch.cuda.synchronize()
    if min_timed_s > 0:
        # short steps: enough of them for the clock sampler (100 ms period) to
        # see the timed region; the same count on every rank
        per = (time.perf_counter() - t_w) / max(warmup, 1)
        steps = int(R.max(float(max(steps, min(200, int(min_timed_s / max(per, 1e-6)) + 1)))))

    # ---- device-resident throughput (value), with live per-kernel timing
    dec.profile(True)
    kernel_ms = {}
    launches = 0
    clk_p, clk_f = sample_clocks_start(local)
    R.barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(steps):
        dec.decode_batch(llr_d, code_id=cid_d, out=out)
        launches += dec.last_launches()
        per = {}  # launches of one pass (an adaptive rung may issue two) summed
        for kd, l, ms in dec.last_kernel_ms():
            per[(kd, l)] = per.get((kd, l), 0.0) + ms
        for k, ms in per.items():
            kernel_ms.setdefault(k, []).append(ms)
    ev1.record(stream)
    torch.cuda.synchronize()
    R.barrier()
    clocks = sample_clocks_stop(clk_p, clk_f)
    dec.profile(False)
    elapsed = R.max(ev0.elapsed_time(ev1) / 1e3)
    ms_per_step = elapsed / steps * 1e3
    value = bits_per_step * ws * steps / elapsed / 1e9

    # ---- per-frame device decode latency (pl_frame_latency; the reference
    # times every decode() call, sim.cpp:54-61), one extra untimed decode
    lat = torch.zeros(F, dtype=torch.int32, device=f"cuda:{local}")
    dec.frame_latency(lat)
    dec.decode_batch(llr_d, code_id=cid_d, out=out)
    torch.cuda.synchronize()
    dec.frame_latency(None)
    lat_us = lat.cpu().numpy().astype(np.float64) / 1e3
    del lat

    # ---- error counts of the batch, reduced over ranks (sim.cpp:66-71)
    pay = out["payload"].cpu().numpy()
    esc = out["esc"].cpu().numpy()
    crc_ok = out["crc_ok"].cpu().numpy()
    metric = out["metric"].cpu().numpy()
    counts = Counters()
    counts.add_batch(np.unpackbits(pay, axis=1), info, esc, ks if cid is not None else None)
    counts = all_reduce_counters(counts, device=R.red_dev if R.group else None)

    # ---- end to end through the public API with host buffers (pl_decode_host)
    host_out = {
        "payload": torch.empty((F, dec.payload_stride), dtype=torch.uint8).pin_memory(),
        "codeword": None,
        "crc_ok": torch.empty(F, dtype=torch.uint8).pin_memory(),
        "esc": torch.empty(F, dtype=torch.uint8).pin_memory(),
        "metric": torch.empty(F, dtype=torch.float32).pin_memory(),
    }
    esz = esize(wl)
    if cid is not None:
        # mixed codes: packed variable-length frames (pl_decode_host_packed),
        # each frame's own n LLRs cross the host link
        pk, off = dec.pack_batch(llr_np, cid)
        pk_h = torch.from_numpy(pk).pin_memory()
        off_h = torch.from_numpy(off).pin_memory()
        e2e_call = lambda: dec.decode_host_packed_into(pk_h, off_h, host_out, cid_h)  # noqa: E731
        h2d = pk.nbytes + off.nbytes + F * 4
        e2e_api = "pl_decode_host_packed"
    else:
        e2e_call = lambda: dec.decode_host_into(llr_h, host_out, cid_h)  # noqa: E731
        h2d = F * dec.llr_stride * esz
        e2e_api = "pl_decode_host"
    e2e_call()
    R.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_call()
    e2e_s = R.max(time.perf_counter() - t0)
    e2e_value = bits_per_step * ws * e2e_steps / e2e_s / 1e9
    d2h = F * (dec.payload_stride + 1 + 1 + 4)
    e2e_same = bool(payload_rows_equal(host_out["payload"].numpy(), pay, codes, cid)
                    and (host_out["esc"].numpy() == esc).all())

    # ---- per-kernel roofline fractions (live CUDA-event durations)
    freq = np.bincount(cid, minlength=len(codes)) / F if cid is not None else np.ones(1)
    bytes_per_frame = float(sum(f * (c.n * esz + (c.payload_size + 7) // 8 + 6)
                                for f, c in zip(freq, codes)))
    sm_count = torch.cuda.get_device_properties(local).multi_processor_count
    clk = (peaks.get("sm_max_mhz") or 1965.0) * 1e6
    lane_peak = sm_count * 128 * clk  # one element-op per lane per clock
    issue_peak = sm_count * 4 * clk  # warp-instructions per second (4 schedulers per SM)
    hbm_peak = peaks["hbm_gbs"]
    nc = ncu_counters(wl)
    kernels = {}
    for (kd, l), v in sorted(kernel_ms.items(), key=lambda kv: -sum(kv[1])):
        s = float(np.mean(v)) / 1e3
        one_pass = kd == "sc" or wl.kind in ("ca_sscl", "sscl", "scl")
        nfr = F if one_pass else int((esc >= l).sum())
        ops = float(sum(f * schedule_work(c, wl.kind, l, wl.pruning, sc=(kd == "sc"))
                        for f, c in zip(freq, codes)))
        e = {"ms": s * 1e3, "share_of_step": s * 1e3 / ms_per_step, "frames": nfr,
             "hbm_achieved_gbs": bytes_per_frame * nfr / s / 1e9,
             "hbm_frac": bytes_per_frame * nfr / s / 1e9 / hbm_peak,
             "element_ops_per_frame": ops, "element_op_frac": ops * nfr / s / lane_peak}
        c = (nc or {}).get("kernels", {}).get(f"{kd}_L{l}")
        if c:
            sc = F / nc["frames"]  # the capture decoded the default batch of the same seed
            e.update({
                "issue_frac": c["warp_inst"] * sc / s / issue_peak,
                "warp_inst_per_frame": c["warp_inst"] * sc / max(nfr, 1),
                "dram_bytes_per_frame": c["dram_bytes"] * sc / max(nfr, 1),
                "dram_frac": c["dram_bytes"] * sc / s / 1e9 / hbm_peak,
                "ncu_issue_active_pct": c["issue_active_pct"], "ncu_alu_pipe_pct": c["alu_pipe_pct"],
                "ncu_smem_bank_conflict_pct": 100.0 * c["smem_bank_conflicts"] / max(c["smem_wavefronts"], 1),
                "kernel": c["kernel"]})
        kernels[f"{kd}_L{l}"] = e
    all_kernel_s = sum(sum(v) for v in kernel_ms.values()) / 1e3 / steps

    # the dominant kernel's roofline: the binding unit of the launch (issue
    # slots for the ALU-bound list kernels, HBM for a DRAM-bound pass)
    dkey = next(iter(kernels))
    d = kernels[dkey]
    per_launch_s = d["ms"] / 1e3
    if "issue_frac" in d and d["issue_frac"] >= d.get("dram_frac", 0.0):
        roof = {"bound": "issue", "achieved": d["issue_frac"] * issue_peak / 1e9,
                "peak": issue_peak / 1e9, "unit": "Gwarp-inst/s", "frac": d["issue_frac"]}
    else:
        roof = {"bound": "hbm", "achieved": d["hbm_achieved_gbs"], "peak": hbm_peak,
                "unit": "GB/s", "frac": d["hbm_frac"]}
    roof.update({
        "kernel": d.get("kernel", dkey), "key": dkey,
        "traffic": d["dram_bytes_per_frame"] * d["frames"] if "dram_bytes_per_frame" in d else None,
        "traffic_frac": d.get("dram_frac"),
        "algorithmic_bytes_per_frame": bytes_per_frame,
        "hbm_algorithmic": {"achieved": d["hbm_achieved_gbs"], "peak": hbm_peak, "unit": "GB/s",
                            "frac": d["hbm_frac"], "peak_source": peak_src},
        "element_op_frac": d["element_op_frac"], "element_ops_per_frame": d["element_ops_per_frame"],
        "launch_ms": per_launch_s * 1e3,
        "counters_source": (nc or {}).get("source"),
    })
    fields = {
        "value": value, "unit": "Gb/s", "ms_per_step": ms_per_step, "steps": steps,
        "warmup": warmup, "dtype": dtype_of(wl), "config": common_config(wl, F, ws),
        "fer": counts.fer(), "frames_counted": counts.frames, "frame_errors": counts.frame_errors,
        "bit_errors": counts.bit_errors, "esc_mean": counts.esc_sum / max(counts.frames, 1),
        # frames per final list size (rank 0's batch): the work each rung sees
        "esc_hist": {int(v): int(c) for v, c in zip(*np.unique(esc, return_counts=True))},
        "gpu_launches": int(launches),
        # rank 0's batch: device time from a frame's first to its last pass
        # output, summed over its passes (a batch of F frames in flight)
        "frame_latency_us": {"mean": float(lat_us.mean()), "p50": float(np.percentile(lat_us, 50)),
                             "p99": float(np.percentile(lat_us, 99)), "max": float(lat_us.max())},
        "kernels": kernels,
        "kernel_share_of_step": all_kernel_s * 1e3 / ms_per_step,
        "roofline": roof,
        "clocks": clocks,
        "e2e": {"value": e2e_value, "unit": "Gb/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "steps": e2e_steps, "api": e2e_api,
                "outputs_equal_device_path": e2e_same},
    }
    state = {"codes": codes, "cid": cid, "ks": ks, "llr": llr_np, "payload": pay, "esc": esc,
             "crc_ok": crc_ok, "metric": metric}
    del llr_d, llr_h, out, host_out, dec
    torch.cuda.empty_cache()
    return fields, state


def payload_rows_equal(a, b, codes, cid):
    """Every frame's own payload bytes equal (mixed batches: rows are as wide
    as the widest code, the bytes past a frame's payload are not written)."""
    n = a.shape[0]
    for i, c in enumerate(codes):
        rows = np.arange(n) if cid is None else np.flatnonzero(cid[:n] == i)
        w = (c.payload_size + 7) // 8
        if not np.array_equal(a[rows, :w], b[rows, :w]):
            return False
    return True


def parity_and_cpu(wl, st, S, nthr, time_it):
    """The compiled reference on the first S frames of the step's batch
    (identical LLR bytes): per-frame parity of payload, crc_ok, escalation
    and metric; the reference's decode time when `time_it`."""
    from oracle import oracle as O

    codes = [(c.n, c.k, c.crc.raw() if c.crc else "", c.frozen) for c in st["codes"]]
    cid = st["cid"][:S] if st["cid"] is not None else None
    r, dt = reference_decode(O, codes, cid, st["llr"][:S], wl, nthr)
    # each frame's own payload bytes (mixed batches: rows are as wide as the widest code)
    bad_pay = np.zeros(S, bool)
    for i, c in enumerate(st["codes"]):
        rows = np.arange(S) if cid is None else np.flatnonzero(cid == i)
        w = (c.payload_size + 7) // 8
        bad_pay[rows] = (st["payload"][rows, :w] != r["payload"][rows, :w]).any(1)
    mism = (bad_pay | (st["crc_ok"][:S] != r["crc_ok"]) | (st["esc"][:S] != r["esc"])
            | (st["metric"][:S] != r["metric"].astype(np.float32)))
    par = {"frames": int(S), "mismatching_frames": int(mism.sum()),
           "fields": "payload, crc_ok, esc, metric (bit-exact)", "against": "oracle/_ref"}
    cpu = None
    if time_it:
        cpu = {"value": float(st["ks"][:S].sum()) / dt / 1e9, "unit": "Gb/s", "cores": nthr,
               "kind": "reference",
               "sample": f"first {S} frames of the step's batch, FrameDecoder<R> per thread "
                         f"({dt:.1f} s wall, {dt * nthr:.0f} core-s)"}
    return par, cpu, dt


def fit_frames(wl, F, R):
    """Multi-rank runs: every rank stages its whole batch in host memory (the
    generated array and, transiently, its pinned copy beside it).  When N such
    stagings would not fit the box's available memory the per-rank batch
    shrinks (all ranks alike: the smallest proposal wins; it stays far above
    the L2 and is what `config.frames_per_gpu` reports)."""
    if R.ws == 1:
        return F
    fit = F
    try:
        import psutil
        per_frame = wl.n * esize(wl) * 2.5
        cap = int(psutil.virtual_memory().available * 0.6 / R.ws / per_frame)
        if cap < F:
            fit = max(4096, cap - cap % 4096)
    except Exception:  # noqa: BLE001
        pass
    return int(-R.max(-float(fit)))


def extra_list(args, ws):
    ex = args.extra if args.extra is not None else (EXTRA_DEFAULT if ws == 1 else EXTRA_DEFAULT_MULTI)
    return [] if ex in ("", "none") else [w for w in ex.split(",") if w != args.workload]


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args)
    if args.impl == "reference":
        return run_reference(args)
    if args.dry_run:
        return run_dry(args)
    from paper_1710_08314_b200.workload import WORKLOADS

    R = Ranks(args)
    ws, rank = R.ws, R.rank
    peaks, peak_src = measured_peaks()
    wl = WORKLOADS[args.workload]
    F = fit_frames(wl, args.frames or wl.frames, R)
    warmup = max(args.warmup, 3)
    e2e_steps = args.e2e_steps or max(3, min(args.steps, 10))
    fields, st = measure(wl, F, args.steps, warmup, e2e_steps, R, peaks, peak_src)
    result = {"metric": METRIC, **fields, "n_gpus": ws, "higher_is_better": True,
              "scaling": "weak", "vs_baseline": None, "data": DATA}

    # ---- CPU baseline + parity: the reference decoder on this box's cores
    nthr = os.cpu_count() or 1
    if rank == 0 and not args.no_cpu:
        try:
            from oracle import oracle as O  # noqa: F401
            if ws == 1:
                # bounded sample: a probe of cpu_sample/4 frames sets the size so
                # the timed run is ~20 core-seconds of reference decoding
                S = min(max(args.cpu_sample // 4, 256), F)
                _, _, dt0 = parity_and_cpu(wl, st, S, nthr, False)
                S = int(min(F, max(args.cpu_sample, S * 20.0 / max(dt0 * nthr, 1e-6))))
                S = max(256, S - S % 256)
            else:
                S = min(args.parity_sample, F)
            par, cpu, _ = parity_and_cpu(wl, st, S, nthr, ws == 1)
            result["parity_vs_reference"] = par
            if cpu:
                result["cpu_baseline"] = cpu
        except Exception as e:  # noqa: BLE001
            result["cpu_baseline"] = {"value": None, "unit": "Gb/s", "cores": 0, "kind": "reference",
                                      "sample": f"unavailable: {e}"}
    del st

    # ---- further BASELINE configs, same measurements (driver-run evidence)
    extras = extra_list(args, ws)
    if extras:
        result["workloads"] = []
        for name in extras:
            w2 = WORKLOADS[name]
            f2, st2 = measure(w2, fit_frames(w2, w2.frames, R), args.extra_steps, warmup, 3, R, peaks,
                              peak_src, min_timed_s=0.4)
            f2 = {"workload": name, **f2}
            if rank == 0 and not args.no_cpu:
                try:
                    S = min(args.parity_sample, len(st2["ks"]))
                    par, cpu, _ = parity_and_cpu(w2, st2, S, nthr, ws == 1)
                    f2["parity_vs_reference"] = par
                    if cpu:
                        f2["cpu_baseline"] = cpu
                except Exception as e:  # noqa: BLE001
                    f2["parity_vs_reference"] = {"unavailable": str(e)}
            del st2
            result["workloads"].append(f2)
    if R.shared:
        result["note"] = f"{ws} ranks shared {torch_device_count()} GPU(s): path exercise only, not a scaling number"
    if R.group:
        result["collectives"] = R.dist.get_backend()
        result["cpu_affinity"] = R.affinity
    result["native_so_loaded"] = mapped_native_libs()
    if rank == 0:
        print(json.dumps(result))
    if R.group:
        R.dist.destroy_process_group()
    return 0


def torch_device_count():
    import torch
    return torch.cuda.device_count()


if __name__ == "__main__":
    sys.exit(main())
