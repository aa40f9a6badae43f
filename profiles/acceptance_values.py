import os, sys; ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import paper_1710_08314_b200 as P
from paper_1710_08314_b200 import sim as S
import test_gpu_acceptance as T
sc = S.SimConfig(code=P.make_code(4096, 2048, P.construct_frozen(4096, 2048, 0.5)), decoder="sc", max_fe=100, max_frames=60000, seed=5001)
ls = S.SimConfig(code=P.make_code(4096, 2048, P.construct_frozen(4096, 2080, 0.5), "32-GZIP"), decoder="ca_sscl", list_size=32, max_fe=100, max_frames=60000, seed=5002)
a=T.find_crossing(T._measure(P,S,sc),2.75,0.25,1e-3); b=T.find_crossing(T._measure(P,S,ls),1.25,0.25,1e-3)
print("c5 sc %.3f ls %.3f gain %.3f"%(a[1],b[1],a[1]-b[1]))
code = P.make_code(2048, 1723, P.construct_frozen(2048, 1755, 0.05), "32-GZIP")
def cfg(prec, rep_max): return S.SimConfig(code=code, decoder="ca_sscl", list_size=8, precision=prec, pruning=P.PruningConfig(rep_max=rep_max), max_fe=100, max_frames=60000, seed=7001)
x=[T.find_crossing(T._measure(P,S,cfg(p,r)),4.0,0.2,1e-3)[1] for p,r in (("f32",0),("i8",8),("i8",0))]
print("c7 f32 %.3f i8cap %.3f (loss %.3f) i8unl %.3f (loss %.3f)"%(x[0],x[1],x[1]-x[0],x[2],x[2]-x[0]))
c4=S.SimConfig(code=P.make_code(2048,1024,P.construct_frozen(2048,1056,0.5),"32-GZIP"),decoder="ca_sscl",precision="f32",max_fe=150,max_frames=400000,seed=4001)
c4.list_size=4; p4=T._point(P,S,c4,2.0); c4.list_size=8; p8=T._point(P,S,c4,2.0)
print("c4 fer4 %.3e (%d/%d) fer8 %.3e (%d/%d) ratio %.3f"%(p4.fer,p4.frame_errors,p4.frames,p8.fer,p8.frame_errors,p8.frames,p8.fer/p4.fer))
# criterion 8 (acceptance.cpp:523-592): the paper's throughput orderings, at batch sizes a GPU needs
HR = 0.05
sp = S.SimConfig(code=P.make_code(2048, 1723, P.construct_frozen(2048, 1723, HR)), decoder="scl", list_size=32, max_frames=32768, max_fe=0, seed=8001)
ti_scl = T._point(P, S, sp, 4.0).ti_mbps; sp.decoder = "sscl"; ti_sscl = T._point(P, S, sp, 4.0).ti_mbps
ad = S.SimConfig(code=P.make_code(2048, 1723, P.construct_frozen(2048, 1755, HR), "32-GZIP"), list_size=8, max_frames=1 << 20, max_fe=0, seed=8002)
ad.decoder = "pa_sscl"; pa = T._point(P, S, ad, 4.0); ad.decoder = "fa_sscl"; fa = T._point(P, S, ad, 4.0)
qa = S.SimConfig(code=ad.code, decoder="fa_sscl", list_size=8, max_frames=1 << 20, max_fe=0, seed=8003)
f32 = T._point(P, S, qa, 4.5); qa.precision = "i8"; qa.pruning = P.PruningConfig(rep_max=8); q8 = T._point(P, S, qa, 4.5)
print("c8 sscl/scl(L=32) %.0f/%.0f = %.2fx (>= 3); fa %.0f >= pa %.0f Mb/s at 4.0 dB; worst frame latency fa %.0f >= pa %.0f us; adaptive 8-bit %.0f >= float %.0f Mb/s at 4.5 dB"
      % (ti_sscl, ti_scl, ti_sscl / ti_scl, fa.ti_mbps, pa.ti_mbps, fa.lat_worst_us, pa.lat_worst_us, q8.ti_mbps, f32.ti_mbps))
