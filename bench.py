#!/usr/bin/env python
"""Benchmark: decoded information throughput (Gb/s) of the B200 polar decoder.

Default workload = BASELINE.json configs[1]: N=2048, K=1723 (+CRC-32 GZIP),
GA frozen set @4.5 dB, CA-SCL L=8 with R0/R1/REP_8-/SPC4 pruning, int8 LLRs
(x4, saturated to +-127) from BPSK-AWGN at 3.5 dB, 262 144 frames per GPU.
One step = one decode of that batch (inputs resident in HBM for `value`;
host buffers with the copies inside the timed region for `e2e`).
`--workload` selects the other BASELINE configs (cfg0, cfg2_{2.5,3.5,4.5},
cfg3 mixed-MCS, cfg4_L{8,16,32}).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg1]
  python bench.py --impl reference ...   # the reference's own CPU decoder
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decoded info throughput (Gb/s) N=2048 K=1723"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="cfg1")
    ap.add_argument("--frames", type=int, default=0, help="override frames per GPU")
    ap.add_argument("--e2e-steps", type=int, default=0)
    ap.add_argument("--cpu-sample", type=int, default=16384)
    ap.add_argument("--ref-sample", type=int, default=16384)
    ap.add_argument("--no-cpu", action="store_true")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


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


def kernel_counters(wl, key, frames):
    """ncu counters of this workload's pass kernel `key` (sc_L1 / list_L<l>),
    per launch of the default batch (profiles/traffic.py, from one committed
    ncu capture per workload); counts scale with the batch size.  None if
    absent."""
    try:
        with open(os.path.join(ROOT, "profiles", "r01_traffic.json")) as fh:
            t = json.load(fh)[wl.name]
        c = dict(t["kernels"][key])
    except (OSError, KeyError, ValueError):
        return None
    s = frames / t["frames"]
    for k in ("dram_bytes", "dram_read_bytes", "dram_write_bytes", "warp_inst"):
        c[k] *= s
    c["source"] = t["source"]
    return c


def common_config(wl, frames_per_gpu, ws):
    """The config both arms report (the driver compares like with like)."""
    esz = {"f32": 4, "i16": 2}.get(wl.precision, 1)
    return {**wl.describe(), "frames_per_gpu": frames_per_gpu,
            "global_frames": frames_per_gpu * ws, "parallelism": f"frame-range shards x{ws}",
            "l2": "inputs larger than L2 (%.0f MB per GPU per step)" % (frames_per_gpu * wl.n * esz / 1e6)}


def reference_decode(O, codes, cid, llr, wl, nthr):
    """The compiled reference FrameDecoder<R> over a batch (per code for
    mixed batches); returns payload/crc_ok/esc/metric arrays and the seconds
    spent decoding."""
    nf = llr.shape[0]
    pb = max((c.payload_size + 7) // 8 for c in codes)
    out = {"payload": np.zeros((nf, pb), np.uint8), "crc_ok": np.zeros(nf, np.uint8),
           "esc": np.zeros(nf, np.uint8), "metric": np.zeros(nf, np.float64)}
    secs = 0.0
    groups = [(0, np.arange(nf))] if cid is None else [(i, np.flatnonzero(cid == i)) for i in range(len(codes))]
    for i, rows in groups:
        if rows.size == 0:
            continue
        c = codes[i]
        ref = O.Reference(c.n, c.k, c.frozen, c.crc.raw() if c.crc else "", wl.kind, wl.l,
                          wl.precision, wl.pruning.as_tuple())
        x = np.ascontiguousarray(llr[rows, : c.n])
        t0 = time.perf_counter()
        r = ref.decode(x, nthr)
        secs += time.perf_counter() - t0
        out["payload"][rows, : r.payload.shape[1]] = r.payload
        out["crc_ok"][rows], out["esc"][rows], out["metric"][rows] = r.crc_ok, r.esc, r.metric
    return out, secs


def run_reference(args):
    """The reference's own CPU decoder (oracle/_ref: FrameDecoder<R> compiled
    from /root/reference/proj), all host threads, bounded sample per step."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    from paper_1710_08314_b200.workload import WORKLOADS, make_batch
    wl = WORKLOADS[args.workload]
    try:
        from oracle import oracle as O
        O.Reference.lib()
    except Exception as e:  # noqa: BLE001
        print(json.dumps({"impl": "reference", "unavailable": f"oracle/_ref not loadable: {e}"}))
        return 0
    nthr = os.cpu_count() or 1
    nf = args.ref_sample
    codes, cid, info, ks, llr = make_batch(wl, 0, nf, nthreads=nthr)
    w = max(nthr, nf // 8)
    reference_decode(O, codes, cid[:w] if cid is not None else None, llr[:w], wl, nthr)  # warm-up
    secs = 0.0
    for _ in range(args.steps):
        secs += reference_decode(O, codes, cid, llr, wl, nthr)[1]
    dt = secs / args.steps
    gbps = float(ks.sum()) / dt / 1e9
    out = {
        "impl": "reference", "metric": METRIC, "value": gbps, "unit": "Gb/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": dtype_of(wl),
        "data": "synthetic: BPSK-AWGN frames keyed by (seed 42, global frame index), FrameRng semantics",
        "config": common_config(wl, args.frames or wl.frames, ws),
        "reference_sample_frames_per_step": nf,
        "cpu_baseline": {"value": gbps, "unit": "Gb/s", "cores": nthr, "kind": "reference",
                         "sample": f"{nf} frames of {wl.name} per step, FrameDecoder<R> per thread"},
        "e2e": {"value": gbps, "unit": "Gb/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out))
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    ws, rank, local = dist_env()
    import torch
    import torch.distributed as dist

    ndev = torch.cuda.device_count()
    shared = ws > ndev  # more ranks than GPUs: only for exercising the path
    if ws > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    local = local % ndev
    torch.cuda.set_device(local)
    import paper_1710_08314_b200 as P
    from paper_1710_08314_b200.shard import Counters, all_reduce_counters, frame_range
    from paper_1710_08314_b200.workload import WORKLOADS, make_batch, schedule_work

    wl = WORKLOADS[args.workload]
    F = args.frames or wl.frames
    frame0, _ = frame_range(rank, ws, F)  # weak scaling: each rank its own global frame range
    codes, cid, info, ks, llr_np = make_batch(wl, frame0, F,
                                              nthreads=max(1, (os.cpu_count() or 1) // ws))
    llr_h = torch.from_numpy(llr_np).pin_memory()
    llr_d = llr_h.cuda(local)
    cid_h = torch.from_numpy(cid).pin_memory() if cid is not None else None
    cid_d = cid_h.cuda(local) if cid is not None else None
    dec = P.FrameDecoder(codes, wl.kind, wl.l, wl.precision, wl.pruning, device=local)
    out = dec.alloc_outputs(F)
    stream = torch.cuda.current_stream(local)
    bits_per_step = float(ks.sum())

    def barrier():
        if ws > 1:
            dist.barrier()

    red_dev = "cpu" if shared else f"cuda:{local}"

    def max_over_ranks(x):
        if ws == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    warmup = max(args.warmup, 3)
    for _ in range(warmup):
        dec.decode_batch(llr_d, code_id=cid_d, out=out)
    torch.cuda.synchronize()

    # ---- device-resident throughput (value), with live per-kernel timing
    dec.profile(True)
    kernel_ms = {}
    launches = 0
    clk_p, clk_f = sample_clocks_start(local)
    barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        dec.decode_batch(llr_d, code_id=cid_d, out=out)
        launches += dec.last_launches()
        per = {}  # launches of one pass (an adaptive rung may issue two) summed
        for kd, l, ms in dec.last_kernel_ms():
            per[(kd, l)] = per.get((kd, l), 0.0) + ms
        for k, ms in per.items():
            kernel_ms.setdefault(k, []).append(ms)
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clocks = sample_clocks_stop(clk_p, clk_f)
    dec.profile(False)
    elapsed = max_over_ranks(ev0.elapsed_time(ev1) / 1e3)
    ms_per_step = elapsed / args.steps * 1e3
    value = bits_per_step * ws * args.steps / elapsed / 1e9

    # ---- error counts of the batch, reduced over ranks (sim.cpp:66-71)
    pay = out["payload"].cpu().numpy()
    esc = out["esc"].cpu().numpy()
    counts = Counters()
    counts.add_batch(np.unpackbits(pay, axis=1), info, esc, ks if cid is not None else None)
    counts = all_reduce_counters(counts, device=red_dev if ws > 1 else None)

    # ---- end to end through the public API with host buffers (pl_decode_host)
    e2e_steps = args.e2e_steps or max(3, min(args.steps, 10))
    host_out = {
        "payload": torch.empty((F, dec.payload_stride), dtype=torch.uint8).pin_memory(),
        "codeword": None,
        "crc_ok": torch.empty(F, dtype=torch.uint8).pin_memory(),
        "esc": torch.empty(F, dtype=torch.uint8).pin_memory(),
        "metric": torch.empty(F, dtype=torch.float32).pin_memory(),
    }
    esz = {"f32": 4, "i16": 2}.get(wl.precision, 1)
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
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_call()
    e2e_s = max_over_ranks(time.perf_counter() - t0)
    e2e_value = bits_per_step * ws * e2e_steps / e2e_s / 1e9
    d2h = F * (dec.payload_stride + 1 + 1 + 4)

    # ---- roofline of the dominant kernel (live CUDA-event durations)
    peaks, peak_src = measured_peaks()
    (dkind, dl), dms = max(kernel_ms.items(), key=lambda kv: sum(kv[1]))
    per_launch_s = float(np.mean(dms)) / 1e3
    one_pass = dkind == "sc" or wl.kind in ("ca_sscl", "sscl", "scl")
    n_launch_frames = F if one_pass else int((esc >= dl).sum())
    # algorithmic bytes / element-ops per frame, averaged over the batch's codes
    freq = np.bincount(cid, minlength=len(codes)) / F if cid is not None else np.ones(1)
    bytes_per_frame = float(sum(f * (c.n * esz + (c.payload_size + 7) // 8 + 6)
                                for f, c in zip(freq, codes)))
    ops_per_frame = float(sum(f * schedule_work(c, wl.kind, dl, wl.pruning, sc=(dkind == "sc"))
                              for f, c in zip(freq, codes)))
    achieved_gbs = bytes_per_frame * n_launch_frames / per_launch_s / 1e9
    sm_count = torch.cuda.get_device_properties(local).multi_processor_count
    clk = (peaks.get("sm_max_mhz") or 1965.0) * 1e6
    lane_peak = sm_count * 128 * clk
    lane_achieved = ops_per_frame * n_launch_frames / per_launch_s
    all_kernel_s = sum(sum(v) for v in kernel_ms.values()) / 1e3

    kc = kernel_counters(wl, f"{dkind}_L{dl}", F)
    issue_peak = sm_count * 4 * clk  # warp-instructions per second (4 schedulers per SM)
    result = {
        "metric": METRIC,
        "value": value, "unit": "Gb/s", "n_gpus": ws, "steps": args.steps,
        "warmup": warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": dtype_of(wl),
        "data": "synthetic: BPSK-AWGN frames keyed by (seed 42, global frame index), FrameRng semantics",
        "config": common_config(wl, F, ws),
        "fer": counts.fer(), "frame_errors": counts.frame_errors, "bit_errors": counts.bit_errors,
        "esc_mean": counts.esc_sum / max(counts.frames, 1),
        # frames per final list size (rank 0's batch): the work each rung sees
        "esc_hist": {int(v): int(c) for v, c in zip(*np.unique(esc, return_counts=True))},
        "gpu_launches": int(launches),
        "kernel_ms": {f"{k[0]}_L{k[1]}": float(np.mean(v)) for k, v in kernel_ms.items()},
        "kernel_share_of_step": all_kernel_s / elapsed if ws == 1 else None,
        "roofline": {"bound": "hbm", "achieved": achieved_gbs, "peak": peaks["hbm_gbs"],
                     "unit": "GB/s", "frac": achieved_gbs / peaks["hbm_gbs"],
                     "traffic": kc["dram_bytes"] if kc else None,
                     "traffic_source": kc["source"] if kc else None,
                     # measured DRAM bytes of the launch / its live duration
                     "traffic_frac": (kc["dram_bytes"] / per_launch_s / 1e9 / peaks["hbm_gbs"]) if kc else None,
                     "kernel": f"decode_kernel<{dtype_of(wl)}, {dkind}> L={dl}",
                     "bytes_per_frame": bytes_per_frame, "peak_source": peak_src},
        # the binding roofline of this issue-bound path: warp-instructions
        # issued per second (ncu's instruction count of the same launch / the
        # live launch time) against 4 per SM per clock, plus ncu's issue-slot
        # and ALU-pipe utilisation of that launch
        "roofline_issue": None if kc is None else {
            "bound": "issue", "achieved": kc["warp_inst"] / per_launch_s / 1e9,
            "peak": issue_peak / 1e9, "unit": "Gwarp-inst/s",
            "frac": kc["warp_inst"] / per_launch_s / issue_peak,
            "warp_inst_per_frame": kc["warp_inst"] / max(n_launch_frames, 1),
            "ncu_issue_active_pct": kc["issue_active_pct"], "ncu_alu_pipe_pct": kc["alu_pipe_pct"],
            "ncu_smem_bank_conflict_pct": 100.0 * kc["smem_bank_conflicts"] / max(kc["smem_wavefronts"], 1),
            "element_ops_per_frame": ops_per_frame,
            "element_op_frac": lane_achieved / lane_peak,
            "source": kc["source"]},
        "clocks": clocks,
        "e2e": {"value": e2e_value, "unit": "Gb/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "steps": e2e_steps, "api": e2e_api},
    }

    # ---- CPU baseline: the reference decoder on this box's cores (rank 0, N=1)
    if rank == 0 and ws == 1 and not args.no_cpu:
        try:
            from oracle import oracle as O
            nthr = os.cpu_count() or 1
            # bounded sample: a probe of cpu_sample/4 frames sets the size so
            # the timed run is ~20 core-seconds of reference decoding
            S = min(max(args.cpu_sample // 4, 256), F)
            _, dt0 = reference_decode(O, codes, cid[:S] if cid is not None else None,
                                      llr_np[:S], wl, nthr)
            S = int(min(F, max(args.cpu_sample, S * 20.0 / max(dt0 * nthr, 1e-6))))
            S = max(256, S - S % 256)
            r, dt = reference_decode(O, codes, cid[:S] if cid is not None else None,
                                     llr_np[:S], wl, nthr)
            cpu_gbps = float(ks[:S].sum()) / dt / 1e9
            pb = r["payload"].shape[1]
            mism = ((pay[:S, :pb] != r["payload"]).any(1) | (out["crc_ok"].cpu().numpy()[:S] != r["crc_ok"])
                    | (esc[:S] != r["esc"])
                    | (out["metric"].cpu().numpy()[:S] != r["metric"].astype(np.float32)))
            result["cpu_baseline"] = {
                "value": cpu_gbps, "unit": "Gb/s", "cores": nthr, "kind": "reference",
                "sample": f"first {S} frames of the step's batch, FrameDecoder<R> per thread "
                          f"({dt:.1f} s wall, {dt * nthr:.0f} core-s)"}
            result["parity_vs_reference"] = {"frames": int(S), "mismatching_frames": int(mism.sum()),
                                             "fields": "payload, crc_ok, esc, metric"}
        except Exception as e:  # noqa: BLE001
            result["cpu_baseline"] = {"value": None, "unit": "Gb/s", "cores": 0, "kind": "reference",
                                      "sample": f"unavailable: {e}"}
    if shared:
        result["note"] = f"{ws} ranks shared {ndev} GPU(s): path exercise only, not a scaling number"
    if rank == 0:
        print(json.dumps(result))
    if ws > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
