"""BASELINE.json workloads and the algorithmic work accounting used by the
roofline.  Harness code: nothing here is on the decode path.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import polar as P

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
            **({"quant_scale": self.scale} if self.precision == "i8" else {}),
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
