#!/usr/bin/env python
"""Per-kernel counters of each bench workload's passes, from one ncu pass per
workload (`profiles/collect_ncu.sh`, its CSVs kept in `<round>_ncu/`):
DRAM bytes, warp-instructions, issue-slot and ALU-pipe utilisation, shared
memory wavefronts / bank conflicts, per launch of the workload's default batch
(the inputs are seeded, so bench.py's launches decode the same frames).

Writes `<round>_traffic.json`, which bench.py reads for the per-kernel
issue / DRAM fractions and `roofline.traffic` of the dominant kernel.

  python profiles/traffic.py [round]     (default r02: profiles/r02_ncu/ -> r02_traffic.json)
"""
import csv
import glob
import json
import os
import re
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from paper_1710_08314_b200.workload import WORKLOADS  # noqa: E402


def kernel_key(name):
    """bench.py's kernel_ms key of a kernel name: sc_L1 / list_L<l>."""
    if "sc_lanes_kernel" in name:
        return "sc_L1"
    m = re.search(r"decode_kernel<[^,]+, (\d+), (\d+), (\d+)(?:, \d+)?>", name)
    kv = int(m.group(1))
    return "sc_L1" if kv == 0 else f"list_L{1 << (kv - 1)}"


RND = sys.argv[1] if len(sys.argv) > 1 else "r02"
out = {}
for path in sorted(glob.glob(os.path.join(HERE, f"{RND}_ncu", "ncu_*.csv"))):
    w = os.path.basename(path)[4:-4]
    rows = [r for r in csv.reader(open(path)) if r]
    rows = rows[next(i for i, r in enumerate(rows) if r[0] == "ID"):]  # skip ==PROF== notes
    hdr = rows[0]
    ix = {k: hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value")}
    launches = {}
    for r in rows[1:]:
        lid = int(r[ix["ID"]])
        d = launches.setdefault(lid, {"kernel": r[ix["Kernel Name"]]})
        d[r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", ""))
    kernels = {}
    best = {}
    for lid in sorted(launches):
        # per pass kernel the longest of its captured launches: an adaptive
        # rung issues two launches of which only one decodes
        d = launches[lid]
        key = kernel_key(d["kernel"])
        if key not in best or d["gpu__time_duration.sum"] > best[key]["gpu__time_duration.sum"]:
            best[key] = d
    for key, d in best.items():
        kernels[key] = {
            "kernel": d["kernel"],
            "dram_bytes": d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"],
            "dram_read_bytes": d["dram__bytes_read.sum"],
            "dram_write_bytes": d["dram__bytes_write.sum"],
            "warp_inst": d["smsp__inst_executed.sum"],
            "issue_active_pct": d["smsp__issue_active.avg.pct_of_peak_sustained_active"],
            "alu_pipe_pct": d["sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"],
            "warps_active_pct": d["sm__warps_active.avg.pct_of_peak_sustained_active"],
            "smem_wavefronts": d["l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"],
            "smem_bank_conflicts": d["l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"],
            "ncu_duration_ns": d["gpu__time_duration.sum"],
        }
    out[WORKLOADS[w].name] = {
        "frames": WORKLOADS[w].frames,
        "kernels": kernels,
        "source": f"profiles/{RND}_ncu/ncu_{w}.csv (profiles/collect_ncu.sh: ncu --metrics, "
                  "the decoding launch of each pass kernel of the workload's default batch)",
    }
json.dump(out, open(os.path.join(HERE, f"{RND}_traffic.json"), "w"), indent=1)
for name, v in out.items():
    for k, d in v["kernels"].items():
        print(f"{name:32s} {k:9s} {d['dram_bytes'] / 1e9:8.2f} GB  {d['warp_inst'] / 1e9:7.2f} Ginst  "
              f"issue {d['issue_active_pct']:5.1f}%  alu {d['alu_pipe_pct']:5.1f}%  "
              f"smem conflicts {d['smem_bank_conflicts'] / max(d['smem_wavefronts'], 1) * 100:4.1f}%")
