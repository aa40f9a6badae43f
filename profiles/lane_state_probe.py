"""How the frame-per-lane SC pass behaves with the state of a list decoder:
SSC on N = 16384 keeps 16 KB of int8 LLR state per frame, like L = 8 paths of
N = 2048 (cfg1), and does 1.27x the f/g work of those (N log N = 229k vs
L N log N = 180k values).  Its time per frame bounds the F/G part of a
frame-per-lane list decoder from above (DESIGN.md §8 item 5).

  python profiles/lane_state_probe.py      (on the GPU box)
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1710_08314_b200 as P  # noqa: E402

for n, k, frames in ((2048, 1723, 1 << 20), (16384, 13784, 1 << 17)):
    for prec in ("i8", "f32"):
        code = P.make_code(n, k, P.construct_frozen_ga(n, k + 32, 4.5, k / n), "32-GZIP")
        dec = P.FrameDecoder(code, "ssc", 1, prec, P.PruningConfig(rep_max=8))
        base = 4096
        _, llr = P.channel(code, 3.5, 42, 0, base, prec, 4.0 if prec == "i8" else 0.0)
        x = torch.from_numpy(np.tile(llr, (frames // base, 1))).cuda()
        out = dec.alloc_outputs(frames)
        for _ in range(2):
            dec.decode_batch(x, out=out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            dec.decode_batch(x, out=out)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        print(f"ssc {prec} N={n}: {frames} frames {ms:.2f} ms -> {ms * 1e3 / frames:.3f} us/frame, "
              f"{ms * 1e6 / frames / (n * np.log2(n)):.4f} ns per f/g value, {k * frames / ms / 1e6:.1f} Gb/s")
