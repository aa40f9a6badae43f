"""Monte-Carlo sweep and report over the GPU decoder.

Mirrors the reference's ``run_montecarlo`` (proj/src/sim.cpp:148-174,
SimConfig / PointStats proj/include/polar/sim.hpp:14-45) and its report
writer (``format_csv_row`` / ``write_report``, proj/src/report.cpp:40-84):

* each Eb/N0 point is ``pl_sim_point``: frames keyed by (seed, global frame
  index) are generated (device Philox channel, or the FrameRng-exact host
  channel), decoded, and compared with their information bits on the device;
  the stop rule is applied at the reference's 1024-frame batch boundaries, so
  with ``channel="host"`` the error counts equal the reference's exactly;
* the sweep loop, its validation and the CSV / table formats are the
  reference's; the timing columns report the GPU (``ti_mbps`` = information
  bits over summed decode-kernel time, ``lat_*`` = per device batch).

Multi-GPU: rank r of ``world`` takes the frame range
[frame0 + r·F/world, frame0 + (r+1)·F/world) of each point (F = max_frames)
and the counts are summed (``shard.all_reduce_counters``); a frame-error
stop rule would need a per-batch exchange, so ``max_fe`` must be 0 then.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import io

from . import _lib as L
from .polar import ConfigError, FrameDecoder, PolarCode, PruningConfig, _raise

COLUMNS = ("ebn0_db", "frames", "bit_errors", "frame_errors", "ber", "fer", "ti_mbps",
           "lat_avg_us", "lat_worst_us", "esc_mean")  # report.cpp:13-16


@dataclasses.dataclass
class SimConfig:
    """sim.hpp:14-29 (psum layout and workers have no GPU meaning; timing is
    always on)."""
    code: PolarCode
    decoder: str = "ssc"
    list_size: int = 8
    precision: str = "f32"
    quant_scale: float = 0.0
    pruning: PruningConfig = dataclasses.field(default_factory=PruningConfig)
    ebn0_min: float = 0.0
    ebn0_max: float = 4.0
    ebn0_step: float = 1.0
    max_frames: int = 10000
    max_fe: int = 100
    seed: int = 42
    channel: str = "device"  # "device" (Philox) or "host" (FrameRng-exact)
    chunk_frames: int = 0
    host_threads: int = 0
    frame0: int = 0
    device: int = 0


@dataclasses.dataclass
class PointStats:
    """sim.hpp:31-42 (+ the escalation sum, for exact multi-rank merges)."""
    ebn0_db: float = 0.0
    frames: int = 0
    bit_errors: int = 0
    frame_errors: int = 0
    ber: float = 0.0
    fer: float = 0.0
    ti_mbps: float = 0.0
    lat_avg_us: float = 0.0
    lat_worst_us: float = 0.0
    esc_mean: float = 0.0
    esc_sum: int = 0


def _validate(cfg: SimConfig):
    # run_montecarlo (sim.cpp:150-158)
    if cfg.ebn0_step <= 0:
        raise ConfigError("Eb/N0 step must be positive")
    if cfg.ebn0_max < cfg.ebn0_min:
        raise ConfigError("Eb/N0 range is empty")
    if cfg.max_frames == 0 and cfg.max_fe == 0:
        raise ConfigError("stop rule is empty: set max frames or target frame errors")
    if cfg.channel not in ("device", "host"):
        raise ConfigError(f"unknown channel {cfg.channel!r}")


def points(cfg: SimConfig):
    """The sweep's Eb/N0 values exactly as run_all enumerates them (sim.cpp:139-144)."""
    i = 0
    while True:
        e = cfg.ebn0_min + float(i) * cfg.ebn0_step
        if e > cfg.ebn0_max + cfg.ebn0_step * 1e-9:
            return
        yield e
        i += 1


def run_point(dec: FrameDecoder, cfg: SimConfig, ebn0_db: float, frame0: int = 0,
              max_frames: int | None = None) -> PointStats:
    c = L.pl_sim_config()
    c.ebn0_db = ebn0_db
    c.seed = cfg.seed
    c.frame0 = frame0
    c.max_frames = cfg.max_frames if max_frames is None else max_frames
    c.max_fe = cfg.max_fe
    c.quant_scale = cfg.quant_scale
    c.channel = L.PL_CHANNEL_HOST if cfg.channel == "host" else L.PL_CHANNEL_DEVICE
    c.host_threads = cfg.host_threads
    c.chunk_frames = cfg.chunk_frames
    out = L.pl_point_stats()
    code = cfg.code.to_c()
    rc = L.lib().pl_sim_point(dec._h, C.byref(code), C.byref(c), C.byref(out))
    if rc:
        _raise(rc, L.last_error(dec._h) or "pl_sim_point failed")
    return PointStats(out.ebn0_db, int(out.frames), int(out.bit_errors), int(out.frame_errors),
                      out.ber, out.fer, out.ti_mbps, out.lat_avg_us, out.lat_worst_us,
                      out.esc_mean, int(out.esc_sum))


def run_montecarlo(cfg: SimConfig, rank: int = 0, world: int = 1, reduce=None) -> list[PointStats]:
    """The sweep.  ``reduce(list_of_ints, op="sum"|"max") -> list_of_ints``
    combines counters over ranks (e.g. a torch.distributed all-reduce) when
    world > 1: the error counts and the per-frame latency sum add up, the
    worst per-frame latency is the maximum."""
    _validate(cfg)
    if world > 1 and (cfg.max_fe or not cfg.max_frames):
        raise ConfigError("multi-rank sweeps need a fixed frame count (max_fe = 0)")
    dec = FrameDecoder(cfg.code, cfg.decoder, cfg.list_size, cfg.precision, cfg.pruning,
                       device=cfg.device)
    out = []
    for e in points(cfg):
        if world > 1:
            a = cfg.max_frames * rank // world
            b = cfg.max_frames * (rank + 1) // world
            p = run_point(dec, cfg, e, cfg.frame0 + a, b - a)
            lat_ns = int(round(p.lat_avg_us * 1e3 * p.frames))
            tot = reduce([p.frames, p.bit_errors, p.frame_errors, p.esc_sum, lat_ns])
            p.frames, p.bit_errors, p.frame_errors, p.esc_sum = (int(x) for x in tot[:4])
            p.lat_avg_us = int(tot[4]) * 1e-3 / p.frames if p.frames else 0.0
            p.lat_worst_us = int(reduce([int(round(p.lat_worst_us * 1e3))], op="max")[0]) * 1e-3
            kf = cfg.code.k * p.frames
            p.ber = p.bit_errors / kf if p.frames else 0.0
            p.fer = p.frame_errors / p.frames if p.frames else 0.0
            p.esc_mean = p.esc_sum / p.frames if p.frames else 0.0
        else:
            p = run_point(dec, cfg, e, cfg.frame0)
        out.append(p)
    return out


def format_csv_row(p: PointStats) -> str:
    """One data row, byte-identical to format_csv_row (report.cpp:40-50)."""
    s = L.pl_point_stats(p.ebn0_db, p.frames, p.bit_errors, p.frame_errors, p.esc_sum, p.ber, p.fer,
                         p.ti_mbps, p.lat_avg_us, p.lat_worst_us, p.esc_mean)
    buf = C.create_string_buffer(512)
    L.lib().pl_format_csv_row(C.byref(s), buf, len(buf))
    return buf.value.decode()


def write_report(stream: io.TextIOBase, fmt: str, meta: list[str], stats: list[PointStats]):
    """'#'-prefixed meta lines, a header, one row per point; "csv" or the
    column-aligned "table" (report.cpp:52-84)."""
    for m in meta:
        stream.write(f"# {m}\n")
    if fmt == "csv":
        stream.write(",".join(COLUMNS) + "\n")
        for p in stats:
            stream.write(format_csv_row(p) + "\n")
        return
    if fmt != "table":
        raise ConfigError(f"unknown report format {fmt!r}")
    rows = [format_csv_row(p).split(",") for p in stats]
    width = [max([len(c)] + [len(r[i]) for r in rows]) for i, c in enumerate(COLUMNS)]
    stream.write("  ".join(c.rjust(width[i]) for i, c in enumerate(COLUMNS)) + "\n")
    for r in rows:
        stream.write("  ".join(v.rjust(width[i]) for i, v in enumerate(r)) + "\n")


def _main(argv=None):
    """A sweep from the command line, e.g. BASELINE configs[4]:

        python -m paper_1710_08314_b200.sim 2048:1024:32-GZIP \\
            --decoder ca_sscl --list-size 32 --ebn0 1.0 4.0 0.5 --frames 16777216

    The code is the first (positional) argument, N:K[:CRC], which keeps the
    options apart from torchrun's own when launched under it.

    Under torchrun each rank takes its frame range of every point and the
    counts are summed with one all-reduce per point (NCCL)."""
    import argparse
    import os
    import sys
    import time

    ap = argparse.ArgumentParser(description=_main.__doc__)
    ap.add_argument("code", nargs="?", default="2048:1024:32-GZIP", help="N:K[:CRC]")
    ap.add_argument("--design", default="ga@2.5", help="ga@<dB> or bhat@<erasure>")
    ap.add_argument("--decoder", default="ca_sscl")
    ap.add_argument("--list-size", type=int, default=8)  # (not --l: torchrun abbreviations)
    ap.add_argument("--precision", default="f32")
    ap.add_argument("--ebn0", type=float, nargs=3, default=[1.0, 4.0, 0.5])
    ap.add_argument("--frames", type=int, default=1 << 20)
    ap.add_argument("--max-fe", type=int, default=0)
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--channel", default="device")
    ap.add_argument("--format", default="csv")
    a = ap.parse_args(argv)
    from . import polar as Pm

    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    reduce = None
    if world > 1:
        import torch
        import torch.distributed as dist

        ndev = torch.cuda.device_count()
        shared = world > ndev  # more ranks than GPUs: exercising the path only
        local = local % ndev
        torch.cuda.set_device(local)
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        red_dev = "cpu" if shared else f"cuda:{local}"

        def reduce(v, op="sum"):
            t = torch.tensor(v, dtype=torch.int64, device=red_dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
            return t.tolist()
    parts = a.code.split(":", 2)
    a.n, a.k, a.crc = int(parts[0]), int(parts[1]), (parts[2] if len(parts) > 2 else "")
    w = Pm.CrcSpec.parse(a.crc).width if a.crc else 0
    kind, val = a.design.split("@")
    fz = (Pm.construct_frozen_ga(a.n, a.k + w, float(val), a.k / a.n) if kind == "ga"
          else Pm.construct_frozen(a.n, a.k + w, float(val)))
    code = Pm.make_code(a.n, a.k, fz, a.crc or None)
    pr = PruningConfig(rep_max=8) if a.precision == "i8" else PruningConfig()
    cfg = SimConfig(code, a.decoder, a.list_size, a.precision, pruning=pr, ebn0_min=a.ebn0[0],
                    ebn0_max=a.ebn0[1], ebn0_step=a.ebn0[2], max_frames=a.frames, max_fe=a.max_fe,
                    seed=a.seed, channel=a.channel, device=local)
    t0 = time.time()
    stats = run_montecarlo(cfg, rank, world, reduce)
    if rank == 0:
        meta = [f"code: N={a.n} K={a.k} crc={a.crc} frozen={a.design}",
                f"decoder: {a.decoder} L={a.list_size} {a.precision}", f"seed: {a.seed}",
                f"channel: {a.channel}", f"gpus: {world}", f"wall_s: {time.time() - t0:.1f}"]
        write_report(sys.stdout, a.format, meta, stats)


if __name__ == "__main__":
    _main()
