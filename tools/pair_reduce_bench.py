"""Fused pair reduce vs collective reduce on an in-process [2,2,1] grid (4
virtual ranks sharing ONE B200, so the 'transfer' is same-device memory):
the time of the NT / TN products of one block backward with the owner
reductions fused into the owner GEMM (default) or run as a separate reduce
(TESS_PAIR_REDUCE=0, set by the caller). Prints one JSON line."""
import json
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2105_14500_b200 as tess  # noqa: E402

q, d = 2, 1
b, s, h, nh = 4, 2048, 4096, 32
grid = tess.GridSpec(q, d)
ctxs = tess.init_local(grid)
dims = tess.LayerDims(b, s, h, nh)
rows, hq = b * s // (q * d), h // q
bf = torch.bfloat16
dev = torch.device("cuda", 0)
steps = int(os.environ.get("STEPS", "5"))
errs, times = [], {}


def run(r):
    try:
        cx = ctxs[r]
        torch.cuda.set_device(0)
        W = [torch.randn(sh, device=dev, dtype=bf) * h ** -0.5
             for sh in ((hq, 3 * hq), (hq, hq), (hq, 4 * hq), (4 * hq, hq))]
        LN = [torch.ones(hq, device=dev), torch.zeros(hq, device=dev),
              torch.ones(hq, device=dev), torch.zeros(hq, device=dev)]
        x = torch.randn(rows, hq, device=dev, dtype=bf)
        dy = torch.randn(rows, hq, device=dev, dtype=bf)
        y, dx = torch.empty_like(x), torch.empty_like(x)
        G = [torch.zeros(t.shape, device=dev) for t in W + LN]
        shard = tess.BlockShardC(*[t.data_ptr() for t in W + LN], 1e-5)
        grads = tess.BlockGradsC(*[t.data_ptr() for t in G])
        st = torch.cuda.Stream(dev)
        sh = st.cuda_stream
        for i in range(steps + 2):
            if i == 2:
                torch.cuda.synchronize()
                t0 = time.time()
            cx.layer_forward("block", "bf16", dims, shard, x.data_ptr(), y.data_ptr(), stream=sh)
            cx.layer_backward("block", "bf16", dims, shard, dy.data_ptr(), dx.data_ptr(), grads,
                              stream=sh)
            cx.stream_join(sh)
        st.synchronize()
        torch.cuda.synchronize()
        times[r] = (time.time() - t0) / steps
    except Exception as e:  # noqa: BLE001
        errs.append(repr(e))


th = [threading.Thread(target=run, args=(r,)) for r in range(grid.size())]
[t.start() for t in th]
[t.join() for t in th]
for c in ctxs:
    c.close()
assert not errs, errs
print(json.dumps({"grid": "[2,2,1] in-process on one GPU", "layer": [b, s, h, nh],
                  "pair_reduce": os.environ.get("TESS_PAIR_REDUCE", "1") != "0",
                  "ms_per_step_max_rank": 1e3 * max(times.values())}))
