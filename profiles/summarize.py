#!/usr/bin/env python
"""Summarise an ncu report of decode_kernel into markdown (for profiles/).

  python profiles/summarize.py gpurun_out/prof.ncu-rep [--frames F] > profiles/rNN_xxx.md

Reads the key SOL / occupancy / issue metrics from the details page and
aggregates the source page (instructions executed, warp-stall samples) by
CUDA source line, so the hot lines are visible without the GUI.
"""
import argparse
import collections
import csv
import io
import subprocess
import sys

csv.field_size_limit(sys.maxsize)

KEYS = [
    "Duration", "Executed Instructions", "Executed Ipc Active", "Issue Slots Busy",
    "Warp Cycles Per Issued Instruction", "Achieved Occupancy", "Theoretical Occupancy",
    "Registers Per Thread", "Dynamic Shared Memory Per Block", "Block Limit Shared Mem",
    "Compute (SM) Throughput", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate",
    "L2 Hit Rate", "Mem Busy", "Avg. Active Threads Per Warp", "Grid Size",
]


def ncu(args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--frames", type=int, default=0)
    ap.add_argument("--top", type=int, default=30)
    ap.add_argument("--src", default="", help="kernels.cu of the profiled revision: "
                    "also bucket instructions by enclosing function")
    a = ap.parse_args()
    det = list(csv.reader(io.StringIO(ncu(["-i", a.rep, "--page", "details", "--csv"]))))
    hdr = det[0]
    mi, vi, ui = hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    ki = hdr.index("Kernel Name")
    print(f"# ncu summary: `{a.rep}`\n")
    print(f"kernel: `{det[1][ki]}`\n")
    print("| metric | value | unit |\n|---|---|---|")
    seen = set()
    for r in det[1:]:
        if r[mi] in KEYS and r[mi] not in seen:
            seen.add(r[mi])
            print(f"| {r[mi]} | {r[vi]} | {r[ui]} |")
            if r[mi] == "Executed Instructions" and a.frames:
                v = float(r[vi].replace(",", ""))
                print(f"| warp-instructions per frame | {v / a.frames:.0f} | inst |")
    raw = list(csv.reader(io.StringIO(ncu(["-i", a.rep, "--page", "raw", "--csv"]))))
    if len(raw) > 2:
        names = raw[0]
        vals = raw[2]
        want = ["dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
                "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
                "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
                "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active"]
        print()
        for w in want:
            if w in names:
                print(f"- `{w}` = {vals[names.index(w)]} {raw[1][names.index(w)]}")
        # issue / pipe utilisation and the stall breakdown (cycles per issued
        # instruction by reason): the issue-bound evidence
        print("\n## issue, pipes, stalls\n")
        print("| metric | value |\n|---|---|")
        for w in ["smsp__issue_active.avg.pct_of_peak_sustained_active",
                  "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
                  "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
                  "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
                  "sm__inst_executed_pipe_adu.avg.pct_of_peak_sustained_active",
                  "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
                  "sm__inst_executed_pipe_cbu.avg.pct_of_peak_sustained_active"]:
            if w in names:
                print(f"| `{w}` | {vals[names.index(w)]} % |")
        st = [(n[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")],
               float(vals[i] or 0)) for i, n in enumerate(names)
              if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio")]
        st = [x for x in sorted(st, key=lambda x: -x[1]) if x[1] >= 0.05]
        if st:
            print("\nstall cycles per issued instruction: " +
                  ", ".join(f"{n} {v:.2f}" for n, v in st))
    mix = list(csv.reader(io.StringIO(ncu(["-i", a.rep, "--page", "raw", "--csv",
                                            "--print-metric-instances", "details"]))))
    if len(mix) > 2 and "sass__inst_executed_per_opcode" in mix[0]:
        v = mix[2][mix[0].index("sass__inst_executed_per_opcode")]
        tot = float(v.split()[0])
        parts = [p.strip().rsplit(":", 1) for p in v[v.index("(") + 1:-1].split(";")]
        print("\nopcode mix (warp-level, % of executed): " +
              ", ".join(f"{o} {float(c) / tot * 100:.1f}" for o, c in parts[:16]))
    src = list(csv.reader(io.StringIO(ncu(["-i", a.rep, "--page", "source", "--csv",
                                            "--print-source", "cuda,sass"]))))
    agg = collections.defaultdict(lambda: [0.0, 0.0])
    text = {}
    hdr = None
    cur = None
    fname = ""
    for r in src:
        if r and r[0] == "File Path":
            fname = r[1].split("/")[-1]
        if r and r[0] == "Line No":
            hdr = r
            ie = hdr.index("Instructions Executed")
            ss = hdr.index("Warp Stall Sampling (All Samples)")
            continue
        if hdr is None or len(r) < len(hdr):
            continue
        if r[0].isdigit():
            cur = (fname, int(r[0]))
            text[cur] = r[1]
        try:
            agg[cur][0] += float(r[ie] or 0)
            agg[cur][1] += float(r[ss] or 0)
        except ValueError:
            pass
    ti = sum(v[0] for v in agg.values()) or 1
    ts = sum(v[1] for v in agg.values()) or 1
    print(f"\n## hot source lines (by warp-stall samples)\n")
    print("| file:line | inst % | stall % | source |\n|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[: a.top]:
        if k is None:
            continue
        s = text.get(k, "").strip().replace("|", "\\|")[:80]
        print(f"| {k[0]}:{k[1]} | {v[0] / ti * 100:.1f} | {v[1] / ts * 100:.1f} | `{s}` |")
    if a.src:
        by_function(agg, ti, ts, a.src)


def by_function(agg, ti, ts, path):
    """Bucket kernels.cu lines by the function whose definition precedes them
    (inlined helpers count where they are written; intrinsic headers apart)."""
    import re
    starts = []
    for i, line in enumerate(open(path), 1):
        m = re.match(r"^(?:__device__|__global__|template <.*> __global__)[^(]*?\b(\w+)\(", line)
        if m:
            starts.append((i, m.group(1)))
    fn = collections.defaultdict(lambda: [0.0, 0.0])
    for k, v in agg.items():
        if k is None:
            continue
        name = k[0]
        if k[0] == "kernels.cu":
            name = "(file scope)"
            for ln, f in starts:
                if ln <= k[1]:
                    name = f
        fn[name][0] += v[0]
        fn[name][1] += v[1]
    print("\n## by function (inlined helpers attributed where written)\n")
    print("| function | inst % | stall % |\n|---|---|---|")
    for k, v in sorted(fn.items(), key=lambda kv: -kv[1][0]):
        if v[0] / ti >= 0.002 or v[1] / ts >= 0.002:
            print(f"| {k} | {v[0] / ti * 100:.1f} | {v[1] / ts * 100:.1f} |")


if __name__ == "__main__":
    main()
