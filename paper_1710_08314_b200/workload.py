"""BASELINE.json workloads and the algorithmic work accounting used by the
roofline.  Harness code: nothing here is on the decode path.
"""
from __future__ import annotations

import os
import re
from dataclasses import dataclass

import numpy as np

from . import polar as P

# GA frozen sets of every workload code in the reference's frozen-file format
# (load_frozen_file, code.cpp:164-185), so the reference arm of bench.py
# builds its codes without this package's library (oracle/frozen/make_frozen.py)
FROZEN_DIR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                          "oracle", "frozen")


def crc_width(crc: str) -> int:
    """Width of a CRC spec text ("32-GZIP", "11:621:0:0:0", ...) without the
    library (crc.cpp:42-84: presets and raw specs both lead with the width)."""
    return int(re.match(r"\d+", crc).group(0)) if crc else 0


def frozen_file(n: int, k: int, crc: str, design_db: float, construction: str = "ga") -> str:
    return os.path.join(FROZEN_DIR, f"{construction}_n{n}_k{k}_c{crc_width(crc)}_d{design_db:g}.frozen")

# op codes of the device schedule (csrc/polar_dev.h)
OP_F, OP_G, OP_H, OP_FROZEN, OP_INFO, OP_R1, OP_REP, OP_SPC = range(8)


@dataclass
class Workload:
    name: str
    n: int
    k: int
    crc: str
    kind: str
    l: int
    precision: str
    pruning: P.PruningConfig
    ebn0_db: float
    frames: int
    scale: float = 0.0
    design_db: float = 4.5
    construction: str = "ga"

    def code_specs(self):
        """[(n, k, crc text, frozen file)] without the library."""
        return [(self.n, self.k, self.crc, frozen_file(self.n, self.k, self.crc, self.design_db,
                                                       self.construction))]

    def code(self) -> P.PolarCode:
        w = P.CrcSpec.parse(self.crc).width if self.crc else 0
        if self.construction == "ga":
            fz = P.construct_frozen_ga(self.n, self.k + w, self.design_db, self.k / self.n)
        else:
            fz = P.construct_frozen(self.n, self.k + w, self.design_db)
        return P.make_code(self.n, self.k, fz, self.crc)

    def describe(self) -> dict:
        return {
            "workload": self.name, "N": self.n, "K": self.k, "crc": self.crc,
            "decoder": self.kind, "L": self.l, "llr": self.precision,
            "pruning": pruning_string(self.pruning), "ebn0_db": self.ebn0_db,
            "frames_per_gpu": self.frames, "frozen": f"{self.construction}@{self.design_db}dB",
            **({"quant_scale": self.scale} if self.precision != "f32" else {}),
        }


def pruning_string(p: P.PruningConfig) -> str:
    """The reference's pruning vocabulary (parse.cpp:123-183)."""
    parts = []
    if p.rate_zero:
        parts.append("R0")
    if p.rate_one:
        parts.append("R1")
    if p.repetition:
        parts.append(f"REP_{p.rep_max}-" if p.rep_max else "REP")
    if p.single_parity:
        parts.append(f"SPC{p.spc_max}+" if p.spc_max == 0 else f"SPC{p.spc_max}")
    return ",".join(parts) or "none"


@dataclass
class MixedWorkload:
    """configs[3]: N in {128..1024} x R in {1/3,1/2,2/3,5/6}, K = floor(N R),
    CRC-11 (0x621) or CRC-24 (0xB2B117) (non-reflected, zero init/xorout,
    SURVEY §B), per-code GA frozen sets at the operating point; the infeasible
    (128, 5/6, CRC-24) pair (K + 24 > 128) is dropped: 31 codes.  Each frame's
    code is a seeded draw keyed by its global index."""
    name: str = "cfg3_mixed_mcs_ca_scl_L8_f32"
    kind: str = "ca_sscl"
    l: int = 8
    precision: str = "f32"
    pruning: P.PruningConfig = P.PruningConfig()
    ebn0_db: float = 3.0
    frames: int = 524288
    scale: float = 0.0
    design_db: float = 3.0
    n: int = 1024  # the widest code (LLR row stride)

    def code_specs(self):
        """[(n, k, crc text, frozen file)] of the 31 codes, without the library."""
        out = []
        for n in (128, 256, 512, 1024):
            for num, den in ((1, 3), (1, 2), (2, 3), (5, 6)):
                k = n * num // den
                for crc in ("11:621:0:0:0", "24:b2b117:0:0:0"):
                    if k + crc_width(crc) > n:
                        continue
                    out.append((n, k, crc, frozen_file(n, k, crc, self.design_db)))
        return out

    def code_list(self):
        out = []
        for n, k, crc, _ in self.code_specs():
            fz = P.construct_frozen_ga(n, k + crc_width(crc), self.design_db, k / n)
            out.append(P.make_code(n, k, fz, crc))
        return out

    def code_ids(self, frame0: int, nframes: int, ncodes: int, seed: int = 42):
        idx = np.arange(frame0, frame0 + nframes, dtype=np.uint64)
        h = (idx * np.uint64(0x9E3779B97F4A7C15)) ^ np.uint64(seed)
        h ^= h >> np.uint64(31)
        h *= np.uint64(0xBF58476D1CE4E5B9)
        h ^= h >> np.uint64(29)
        return (h % np.uint64(ncodes)).astype(np.int32)

    def describe(self) -> dict:
        return {"workload": self.name, "N": "128..1024", "K": "floor(N*R)", "crc": "CRC-11/CRC-24",
                "decoder": self.kind, "L": self.l, "llr": self.precision,
                "pruning": pruning_string(self.pruning), "ebn0_db": self.ebn0_db,
                "frames_per_gpu": self.frames, "frozen": f"ga@{self.design_db}dB per code",
                "codes": 31}


def make_batch(wl, frame0: int, nframes: int, seed: int = 42, nthreads: int = 0):
    """Host inputs for a bench step: (codes, code_id or None, info (F, kmax),
    k per frame, llr (F, stride)), frames keyed by global index."""
    dt = np.float32 if wl.precision == "f32" else np.int8
    if isinstance(wl, MixedWorkload):
        codes = wl.code_list()
        cid = wl.code_ids(frame0, nframes, len(codes), seed)
        nmax = max(c.n for c in codes)
        kmax = max(c.k for c in codes)
        llr = np.zeros((nframes, nmax), dt)
        info = np.zeros((nframes, kmax), np.uint8)
        ks = np.zeros(nframes, np.int32)
        for i, c in enumerate(codes):
            rows = np.flatnonzero(cid == i)
            if rows.size == 0:
                continue
            tl = np.zeros((rows.size, nmax), dt)
            ti = np.zeros((rows.size, kmax), np.uint8)
            P.channel_frames(c, wl.ebn0_db, seed, rows.astype(np.uint64) + np.uint64(frame0), tl, ti,
                             wl.precision, wl.scale, nthreads)
            llr[rows] = tl
            info[rows] = ti
            ks[rows] = c.k
        return codes, cid, info, ks, llr
    code = wl.code()
    info, llr = P.channel(code, wl.ebn0_db, seed, frame0, nframes, wl.precision, wl.scale, nthreads)
    return [code], None, info, np.full(nframes, code.k, np.int32), llr


WORKLOADS = {
    # configs[0]: CA-SCL L=4, float, 4.5 dB, 65 536 frames
    "cfg0": Workload("cfg0_ca_scl_L4_f32", 2048, 1723, "32-GZIP", "ca_sscl", 4, "f32",
                     P.PruningConfig(), 4.5, 65536),
    # configs[1]: CA-SCL L=8, int8 (x4, +-127), REP_8-, 3.5 dB, 262 144 frames
    "cfg1": Workload("cfg1_ca_scl_L8_i8", 2048, 1723, "32-GZIP", "ca_sscl", 8, "i8",
                     P.PruningConfig(rep_max=8), 3.5, 262144, scale=4.0),
    # configs[2]: fully adaptive up to L=32, float, per SNR point
    "cfg2_2.5": Workload("cfg2_fa_scl_L32_f32@2.5dB", 2048, 1723, "32-GZIP", "fa_sscl", 32, "f32",
                         P.PruningConfig(), 2.5, 1048576),
    "cfg2_3.5": Workload("cfg2_fa_scl_L32_f32@3.5dB", 2048, 1723, "32-GZIP", "fa_sscl", 32, "f32",
                         P.PruningConfig(), 3.5, 1048576),
    "cfg2_4.5": Workload("cfg2_fa_scl_L32_f32@4.5dB", 2048, 1723, "32-GZIP", "fa_sscl", 32, "f32",
                         P.PruningConfig(), 4.5, 1048576),
    # configs[3]: mixed MCS, CA-SCL L=8, float, 3 dB, 524 288 frames
    "cfg3": MixedWorkload(),
    # the paper's fixed-point FA-SSCL points: same code as
    # configs[2], L=32 at 4.5 dB, int8 (x4, REP_8-) and int16 (x64)
    "fa_i8_4.5": Workload("fa_scl_L32_i8@4.5dB", 2048, 1723, "32-GZIP", "fa_sscl", 32, "i8",
                          P.PruningConfig(rep_max=8), 4.5, 1048576, scale=4.0),
    "fa_i16_4.5": Workload("fa_scl_L32_i16@4.5dB", 2048, 1723, "32-GZIP", "fa_sscl", 32, "i16",
                           P.PruningConfig(), 4.5, 1048576),
    # configs[4]: N=2048, K=1024 + CRC-32, CA-SCL L in {8,16,32}; one SNR
    # point per bench step (the 1..4 dB sweep: python -m paper_1710_08314_b200.sim)
    "cfg4_L8": Workload("cfg4_ca_scl_L8_f32@2.5dB", 2048, 1024, "32-GZIP", "ca_sscl", 8, "f32",
                        P.PruningConfig(), 2.5, 65536, design_db=2.5),
    "cfg4_L16": Workload("cfg4_ca_scl_L16_f32@2.5dB", 2048, 1024, "32-GZIP", "ca_sscl", 16, "f32",
                         P.PruningConfig(), 2.5, 65536, design_db=2.5),
    "cfg4_L32": Workload("cfg4_ca_scl_L32_f32@2.5dB", 2048, 1024, "32-GZIP", "ca_sscl", 32, "f32",
                         P.PruningConfig(), 2.5, 32768, design_db=2.5),
}


def schedule_work(code: P.PolarCode, kind: str, l: int, pruning: P.PruningConfig, sc: bool = False):
    """Element-ops per frame E(tree, L): sum over branch ops of
    alive * m/2 and over leaf ops of alive * m, with the data-independent alive
    trace alive <- min(l, alive * branching)."""
    kd = P.DecoderKind[kind]
    tree = P.prune_tree(code.frozen, pruning if kd.uses_pruning else P.PruningConfig.none())
    work = 0
    alive = 1

    def walk(i):
        nonlocal work, alive
        kind_, depth, lb, size, left, right = (int(x) for x in tree[i])
        if kind_ == 0:
            work += alive * size // 2
            walk(left)
            work += alive * size // 2
            walk(right)
            work += alive * size // 2
            return
        if sc and kind_ in (4, 6):  # R1 / SPC decoded by full recursion on the SC rung
            work += size * int(np.log2(size)) * 3 // 2 + size
            return
        work += alive * size
        if not sc:
            if kind_ == 2:
                alive = min(l, 2 * alive)
            elif kind_ == 4:
                alive = min(l, 4 * alive)
            elif kind_ in (5, 6):
                alive = min(l, 2 * alive)

    walk(0)
    return work
