#!/usr/bin/env python
"""DRAM traffic per frame of the first decode kernel of each bench workload,
from one ncu pass per workload:

  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \\
      -k regex:decode_kernel -c 1 --csv python bench.py --workload W --steps 1 --warmup 0 --no-cpu

(`r01_traffic_ncu.log` holds the grepped lines).  Writes `r01_traffic.json`,
which bench.py reads for `roofline.traffic` (bytes per launch)."""
import collections
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from paper_1710_08314_b200.workload import WORKLOADS  # noqa: E402

vals = collections.defaultdict(dict)
for line in open(os.path.join(HERE, "r01_traffic_ncu.log")):
    w, metric, v = line.split()
    vals[w][metric] = float(v.strip('"'))
out = {}
for w, m in vals.items():
    frames = WORKLOADS[w].frames
    dram = m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]
    out[WORKLOADS[w].name] = {
        "frames_per_launch": frames,
        "dram_bytes_per_launch": dram,
        "dram_bytes_per_frame": dram / frames,
        "dram_read_bytes": m["dram__bytes_read.sum"],
        "dram_write_bytes": m["dram__bytes_write.sum"],
        "source": "profiles/r01_traffic_ncu.log (ncu --metrics dram__bytes_read.sum,"
                  "dram__bytes_write.sum, first decode_kernel launch)",
    }
json.dump(out, open(os.path.join(HERE, "r01_traffic.json"), "w"), indent=1)
for k, v in out.items():
    print(f"{k:32s} {v['dram_bytes_per_frame']:10.0f} B/frame")
