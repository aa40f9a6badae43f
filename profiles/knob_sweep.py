#!/usr/bin/env python
"""Sweep the launch-placement knobs (PLB_TARGET_WARPS, PLB_SEGMAX) for one
bench workload; prints one line per setting (value or the error tail)."""
import json
import os
import subprocess
import sys

wl = sys.argv[1]
targets = [int(x) for x in sys.argv[2].split(",")]
segs = sys.argv[3].split(",")
for t in targets:
    for s in segs:
        env = {**os.environ, "PLB_TARGET_WARPS": str(t)}
        if s != "auto":
            env["PLB_SEGMAX"] = s
        r = subprocess.run([sys.executable, "bench.py", "--workload", wl, "--steps", "3", "--warmup", "3",
                            "--no-cpu", "--e2e-steps", "1"], capture_output=True, text=True, env=env)
        try:
            d = json.loads(r.stdout.strip().splitlines()[-1])
            print(f"target={t} segmax={s} value={d['value']:.3f} kernel_ms={d['kernel_ms']}", flush=True)
        except Exception:  # noqa: BLE001
            print(f"target={t} segmax={s} FAILED: {(r.stderr or r.stdout).strip().splitlines()[-1:]}", flush=True)
