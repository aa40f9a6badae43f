#!/usr/bin/env python
"""In-process knob sweep on one bench workload (run on the GPU box).

  python profiles/sweep.py <workload> <frames> "K=V,K=V" "K=V" ...

The batch is generated and uploaded once; for every setting the PLB_*
variables are set, a fresh decoder is created (the library reads them at
pl_create), warmed up and timed over 3 decodes with CUDA events; per-pass
kernel times come from pl_profile.  Outputs must be identical for every
setting (the knobs are placement only): a mismatch is printed as DIFF.
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1710_08314_b200 as P  # noqa: E402
from paper_1710_08314_b200.workload import WORKLOADS, make_batch  # noqa: E402

wl = WORKLOADS[sys.argv[1]]
F = int(sys.argv[2]) or wl.frames
codes, cid, info, ks, llr = make_batch(wl, 0, F, nthreads=os.cpu_count() or 1)
x = torch.from_numpy(llr).cuda()
c = torch.from_numpy(cid).cuda() if cid is not None else None
ref = None
for setting in sys.argv[3:]:
    keys = []
    for kv in filter(None, setting.split(",")):
        k, v = kv.split("=")
        os.environ[k] = v
        keys.append(k)
    dec = P.FrameDecoder(codes, wl.kind, wl.l, wl.precision, wl.pruning)
    out = dec.alloc_outputs(F)
    for _ in range(2):
        dec.decode_batch(x, code_id=c, out=out)
    torch.cuda.synchronize()
    dec.profile(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    per = {}
    e0.record()
    for _ in range(3):
        dec.decode_batch(x, code_id=c, out=out)
        for kd, l, ms in dec.last_kernel_ms():
            per[f"{kd}{l}"] = per.get(f"{kd}{l}", 0.0) + ms / 3
    e1.record()
    torch.cuda.synchronize()
    dec.profile(False)
    ms = e0.elapsed_time(e1) / 3
    res = [out[k].cpu().numpy().copy() for k in ("payload", "esc", "metric", "crc_ok")]
    same = "" if ref is None else ("same" if all(np.array_equal(a, b) for a, b in zip(ref, res)) else "DIFF")
    if ref is None:
        ref = res
    gbps = float(ks.sum()) / ms / 1e6
    e2e = ""
    if os.environ.get("SWEEP_E2E"):
        # the host API with pinned buffers (packed frames for mixed codes)
        hp = {"payload": torch.empty((F, dec.payload_stride), dtype=torch.uint8).pin_memory(),
              "crc_ok": torch.empty(F, dtype=torch.uint8).pin_memory(),
              "esc": torch.empty(F, dtype=torch.uint8).pin_memory(),
              "metric": torch.empty(F, dtype=torch.float32).pin_memory()}
        if cid is not None:
            pk, off = dec.pack_batch(llr, cid)
            pk_h, off_h = torch.from_numpy(pk).pin_memory(), torch.from_numpy(off).pin_memory()
            cid_h = torch.from_numpy(cid).pin_memory()
            call = lambda: dec.decode_host_packed_into(pk_h, off_h, hp, cid_h)  # noqa: E731
        else:
            llr_h = torch.from_numpy(llr).pin_memory()
            call = lambda: dec.decode_host_into(llr_h, hp)  # noqa: E731
        call()
        t0 = time.perf_counter()
        for _ in range(3):
            call()
        e2e = f" e2e {float(ks.sum()) * 3 / (time.perf_counter() - t0) / 1e9:7.3f} Gb/s"
    print(f"{setting or 'default':40s} {gbps:8.3f} Gb/s  {ms:8.3f} ms{e2e}  "
          + " ".join(f"{k}={v:.3f}" for k, v in per.items()) + f"  {same}", flush=True)
    for k in keys:
        del os.environ[k]
    del dec, out
