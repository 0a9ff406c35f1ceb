"""LayerNorm fwd+bwd (the `layernorm` layer op, with dgain/dbias) at the
cfg4 per-rank shape: rows 16384 per rank, hidden 12288, bf16. GRID=q,d
(default 2,1: 4 in-process ranks sharing ONE B200, h/q = 6144, the split
path: partials -> row all-reduce -> apply) or 1,1 (the fused single pass).
Prints one JSON line: wall ms per step (max over ranks) and the aggregate
compulsory HBM bytes of all ranks over that time."""
import json
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2105_14500_b200 as tess  # noqa: E402

q, d = [int(v) for v in os.environ.get("GRID", "2,1").split(",")]
h, s, nh = 12288, 2048, 96
rows = 16384
b = rows * d * q // s
grid = tess.GridSpec(q, d, d > q)
ctxs = tess.init_local(grid)
dims = tess.LayerDims(b, s, h, nh)
hq = h // q
bf = torch.bfloat16
dev = torch.device("cuda", 0)
steps = int(os.environ.get("STEPS", "20"))
errs, times, kern = [], {}, {}
bar = threading.Barrier(grid.size())


def run(r):
    try:
        cx = ctxs[r]
        torch.cuda.set_device(0)
        dummy = torch.zeros(8, device=dev, dtype=bf)
        LN = [torch.ones(hq, device=dev), torch.zeros(hq, device=dev),
              torch.ones(hq, device=dev), torch.zeros(hq, device=dev)]
        x = torch.randn(rows, hq, device=dev, dtype=bf)
        dy = torch.randn(rows, hq, device=dev, dtype=bf)
        y, dx = torch.empty_like(x), torch.empty_like(x)
        G = [torch.zeros(8, device=dev) for _ in range(4)] + \
            [torch.zeros(hq, device=dev) for _ in range(4)]
        shard = tess.BlockShardC(*[dummy.data_ptr()] * 4, *[t.data_ptr() for t in LN], 1e-5)
        grads = tess.BlockGradsC(*[t.data_ptr() for t in G])
        st = torch.cuda.Stream(dev)
        sh = st.cuda_stream
        for i in range(steps + 3):
            if i == 3:
                st.synchronize()
                bar.wait()
                t0 = time.time()
            cx.layer_forward("layernorm", "bf16", dims, shard, x.data_ptr(), y.data_ptr(),
                             stream=sh)
            cx.layer_backward("layernorm", "bf16", dims, shard, dy.data_ptr(), dx.data_ptr(),
                              grads, stream=sh)
            cx.stream_join(sh)
        st.synchronize()
        times[r] = (time.time() - t0) / steps
    except Exception as e:  # noqa: BLE001
        errs.append(repr(e))


th = [threading.Thread(target=run, args=(r,)) for r in range(grid.size())]
[t.start() for t in th]
[t.join() for t in th]
for c in ctxs:
    c.close()
assert not errs, errs
ms = 1e3 * max(times.values())
# per rank: fwd read x + write y; bwd read dy, x + write dx (bf16)
nbytes = grid.size() * rows * hq * 2 * 5
print(json.dumps({"grid": grid.to_string(), "rows_per_rank": rows, "width": hq,
                  "ms_per_step_max_rank": ms, "aggregate_gbs": nbytes / (ms * 1e-3) / 1e9}))
