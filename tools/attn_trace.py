"""Phase timeline of the fused attention backward (CTA 0 of the cfg4 shape):
TESS_ATTN_TRACE=1 python tools/attn_trace.py"""
import ctypes as C
import os
import sys

os.environ["TESS_ATTN_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import runpy  # noqa: E402

import paper_2105_14500_b200 as tess  # noqa: E402

sys.argv = ["ncu_step.py"]
runpy.run_path(os.path.join(os.path.dirname(__file__), "ncu_step.py"))
buf = (C.c_longlong * 512)()
tess.lib.tess_debug_attn_trace(buf, 512)
ev = [[buf[e * 64 + t] for t in range(64)] for e in range(8)]
t0 = min(v for row in ev for v in row if v)
names = ["MMA scores(i)", "MMA pds_full(i)", "SM sdp_full(i)", "SM chunk0 done", "SM pds_full", "SM tmem loaded", "MMA sdp_free(i)", "MMA grads(i) out"]
print("tile " + " ".join(f"{n:>18s}" for n in names))
for t in range(int(os.environ.get("TILES", "16"))):
    print(f"{t:4d} " + " ".join(f"{(ev[e][t] - t0) if ev[e][t] else -1:18d}" for e in range(8)))
