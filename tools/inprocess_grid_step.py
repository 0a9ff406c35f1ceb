"""The benchmark's own workload on its target grid, on ONE B200: cfg4 (h 12288,
96 heads, s 2048, b = 4 p) block fwd+bwd on an in-process [q,q,d] grid, one
host thread per virtual rank, all ranks sharing cuda:0 (the in-process
backend: collectives are same-device copies / sum kernels, the NT / TN
reduces fused into the owner GEMMs). It shows the whole [2,2,2] path running
at full size -- partition geometry, every collective, the per-rank CommStats
-- and what the 8 ranks' work costs when serialised on one GPU. It says
nothing about multi-GPU scaling: the GPU is shared, and no NVLink is used.

  GRID=2,2 STEPS=2 python tools/inprocess_grid_step.py   -> one JSON line
"""
import json
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2105_14500_b200 as tess  # noqa: E402

q, d = [int(v) for v in os.environ.get("GRID", "2,2").split(",")]
steps = int(os.environ.get("STEPS", "2"))
h, nh, s = 12288, 96, 2048
grid = tess.GridSpec(q, d, d > q)
p = grid.size()
b = 4 * p
dims = tess.LayerDims(b, s, h, nh)
rows, hq = b * s // (d * q), h // q
bf = torch.bfloat16
dev = torch.device("cuda", 0)
ctxs = tess.init_local(grid)
bar = threading.Barrier(p)
errs, times, stats = [], {}, {}


def run(r):
    try:
        cx = ctxs[r]
        torch.cuda.set_device(0)
        g = torch.Generator(device=dev)
        g.manual_seed(1234 + r)
        W = [(torch.rand(sh, device=dev, generator=g) * 2 - 1).mul_(h ** -0.5).to(bf)
             for sh in ((hq, 3 * hq), (hq, hq), (hq, 4 * hq), (4 * hq, hq))]
        LN = [torch.ones(hq, device=dev), torch.zeros(hq, device=dev),
              torch.ones(hq, device=dev), torch.zeros(hq, device=dev)]
        x = (torch.rand(rows, hq, device=dev, generator=g) * 2 - 1).to(bf)
        dy = (torch.rand(rows, hq, device=dev, generator=g) * 2 - 1).to(bf)
        y, dx = torch.empty_like(x), torch.empty_like(x)
        G = [torch.empty(t.shape, device=dev) for t in W + LN]
        shard = tess.BlockShardC(*[t.data_ptr() for t in W + LN], 1e-5)
        grads = tess.BlockGradsC(*[t.data_ptr() for t in G])
        st = torch.cuda.Stream(dev)
        sh = st.cuda_stream
        for i in range(steps + 1):
            if i == 1:
                st.synchronize()
                bar.wait()
                cx.reset_stats()
                t0 = time.time()
            cx.layer_forward("block", "bf16", dims, shard, x.data_ptr(), y.data_ptr(), stream=sh)
            cx.layer_backward("block", "bf16", dims, shard, dy.data_ptr(), dx.data_ptr(), grads,
                              stream=sh)
            cx.stream_join(sh)
        st.synchronize()
        bar.wait()
        times[r] = (time.time() - t0) / steps
        stats[r] = cx.stats()
        assert torch.isfinite(dx.float()).all() and torch.isfinite(G[2]).all()
    except Exception as e:  # noqa: BLE001
        errs.append(repr(e))


th = [threading.Thread(target=run, args=(r,)) for r in range(p)]
[t.start() for t in th]
[t.join() for t in th]
for c in ctxs:
    c.close()
assert not errs, errs
ms = 1e3 * max(times.values())
flops = 72.0 * b * s * h * h + 12.0 * b * s * s * h
sent = [stats[r]["sent_elements"] // steps for r in range(p)]
print(json.dumps({
    "grid": grid.to_string(), "ranks_sharing_one_gpu": p,
    "layer": {"batch": b, "seq": s, "hidden": h, "heads": nh, "rows_per_rank": rows,
              "hidden_per_rank": hq},
    "wall_ms_per_step_all_ranks": ms,
    "tflops_of_the_whole_grid_on_one_gpu": flops / (ms * 1e-3) / 1e12,
    "sent_elements_per_rank_per_step": sent,
    "note": "virtual ranks share cuda:0; not a scaling number"}))
