#!/usr/bin/env python
"""Cycles per list-decoder op kind of one frame (frame 0), from the
profiling build (PLB_OPTIME: clock64 around every op of frame 0's decode):

  PLB_LIB=paper_1710_08314_b200/libpolar_b200_opt.so python profiles/optime_probe.py

Run alone (1 frame: the latency floor of a small FA rung) and inside a full
batch (the op mix under load).  Not a timing of the product build."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1710_08314_b200 as P  # noqa: E402
from paper_1710_08314_b200 import _lib  # noqa: E402
from paper_1710_08314_b200.workload import WORKLOADS, make_batch  # noqa: E402

NAMES = ["F", "G", "H", "FROZEN", "INFO", "R1", "REP", "SPC"]
lib = _lib.lib()
lib.pl_debug_optime.argtypes = [C.c_void_p, C.c_int]


def probe(name, kind, l, prec, nframes):
    wl = WORKLOADS[name]
    codes, cid, info, ks, llr = make_batch(wl, 0, max(nframes, 1), nthreads=os.cpu_count() or 1)
    dec = P.FrameDecoder(codes, kind, l, prec, wl.pruning)
    x = torch.from_numpy(llr).cuda()
    dec.decode_batch(x)
    torch.cuda.synchronize()
    buf = (C.c_ulonglong * 64)()
    lib.pl_debug_optime(buf, 1)  # reset
    dec.decode_batch(x)
    torch.cuda.synchronize()
    lib.pl_debug_optime(buf, 1)
    cyc = np.array(buf[:32], np.float64)
    cnt = np.array(buf[32:], np.float64)
    tot = cyc.sum()
    print(f"== {name} {kind} L={l} {prec} frames={nframes}: {tot:.0f} cycles for frame 0 "
          f"({tot / 1.965e3:.1f} us at 1965 MHz), {int(cnt.sum())} ops")
    for s in range(16):
        if cnt[s]:
            nm = NAMES[s // 2] + ("+fused" if s & 1 else "")
            print(f"   {nm:14s} ops {int(cnt[s]):5d}  cycles/op {cyc[s] / cnt[s]:8.0f}  share {cyc[s] / tot * 100:5.1f}%")


probe("cfg1", "ca_sscl", 8, "i8", 1)
probe("cfg1", "ca_sscl", 8, "i8", 262144)
probe("cfg2_4.5", "ca_sscl", 2, "f32", 1)
probe("cfg2_4.5", "ca_sscl", 4, "f32", 1)
probe("cfg2_4.5", "ca_sscl", 32, "f32", 1)
probe("cfg0", "ca_sscl", 4, "f32", 65536)
probe("cfg4_L32", "ca_sscl", 32, "f32", 32768)
