import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1710_08314_b200 as P
from paper_1710_08314_b200.workload import WORKLOADS, make_batch
wl = WORKLOADS["cfg2_4.5"]
code = wl.code()
# one-frame passes at every L (ca_sscl), 3 reps
_, llr = P.channel(code, 4.5, 42, 0, 64, "f32")
x = torch.from_numpy(llr).cuda()
for l in (2, 4, 8, 16, 32):
    for nf in (1, 45, 300):
        dec = P.FrameDecoder(code, "ca_sscl", l, "f32", wl.pruning)
        xx = x[:1].repeat(nf, 1).contiguous()
        for _ in range(2): dec.decode_batch(xx)
        torch.cuda.synchronize()
        dec.profile(True)
        dec.decode_batch(xx); torch.cuda.synchronize()
        print(f"L={l:2d} frames={nf:4d} kernel_ms={dec.last_kernel_ms()}", flush=True)
        dec.profile(False)
# FA 4.5 dB per-frame latency by escalation level
codes, cid, info, ks, llr = make_batch(wl, 0, 262144, nthreads=os.cpu_count())
dec = P.FrameDecoder(codes, wl.kind, wl.l, wl.precision, wl.pruning)
xx = torch.from_numpy(llr).cuda()
lat = torch.zeros(xx.shape[0], dtype=torch.int32, device="cuda")
dec.frame_latency(lat)
for _ in range(2): out = dec.decode_batch(xx)
dec.profile(True); out = dec.decode_batch(xx); torch.cuda.synchronize()
print(dec.last_kernel_ms())
t = lat.cpu().numpy().astype(np.int64); e = out["esc"].cpu().numpy()
for v in np.unique(e):
    sel = t[e == v]
    print(f"esc={v:2d} frames={sel.size:7d} lat_us mean={sel.mean()/1e3:9.1f} max={sel.max()/1e3:9.1f}")
