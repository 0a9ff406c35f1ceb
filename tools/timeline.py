"""Kernel timeline of one cfg4 block fwd+bwd at [1,1,1] (torch.profiler /
CUPTI sees libtess's kernels): per-kernel device time, and the idle gaps
between consecutive kernels on the GPU (launch-bound or host-bound stalls).
Prints a summary; writes gpurun_out/timeline.json (chrome trace)."""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2105_14500_b200 as tess  # noqa: E402

h, nh, s, b = 12288, 96, 2048, int(os.environ.get("BATCH", "4"))
dev = torch.device("cuda", 0)
ctx = tess.init_local(tess.GridSpec(1, 1))[0]
rows, hq = b * s, h
bf = torch.bfloat16
W = [torch.randn(sh, device=dev, dtype=bf) * h ** -0.5
     for sh in ((hq, 3 * hq), (hq, hq), (hq, 4 * hq), (4 * hq, hq))]
LN = [torch.ones(hq, device=dev), torch.zeros(hq, device=dev), torch.ones(hq, device=dev),
      torch.zeros(hq, device=dev)]
x, dy = torch.randn(rows, hq, device=dev, dtype=bf), torch.randn(rows, hq, device=dev, dtype=bf)
y, dx = torch.empty_like(x), torch.empty_like(x)
G = [torch.empty(t.shape, device=dev) for t in W + LN]
shard = tess.BlockShardC(*[t.data_ptr() for t in W + LN], 1e-5)
grads = tess.BlockGradsC(*[t.data_ptr() for t in G])
dims = tess.LayerDims(b, s, h, nh)
st = torch.cuda.current_stream().cuda_stream


def step():
    ctx.layer_forward("block", "bf16", dims, shard, x.data_ptr(), y.data_ptr(), stream=st)
    ctx.layer_backward("block", "bf16", dims, shard, dy.data_ptr(), dx.data_ptr(), grads,
                       stream=st)


for _ in range(3):
    step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(2):
        step()
    torch.cuda.synchronize()
os.makedirs("gpurun_out", exist_ok=True)
prof.export_chrome_trace("gpurun_out/timeline.json")
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev = sorted(ev, key=lambda e: e.time_range.start)
agg = collections.defaultdict(lambda: [0.0, 0])
for e in ev:
    a = agg[e.name[:90]]
    a[0] += (e.time_range.end - e.time_range.start) / 1e3
    a[1] += 1
span = (ev[-1].time_range.end - ev[0].time_range.start) / 1e3
busy = sum(a[0] for a in agg.values())
gaps = []
for p, n in zip(ev, ev[1:]):
    g = (n.time_range.start - p.time_range.end) / 1e3
    if g > 0.02:
        gaps.append((g, p.name[:60], n.name[:60]))
print(f"2 steps: span {span:.3f} ms, kernel-busy {busy:.3f} ms, idle {span - busy:.3f} ms")
for n, (ms, k) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:30]:
    print(f"{ms:9.3f} ms x{k:<4d} {n}")
print("largest gaps (ms, after, before):")
for g in sorted(gaps, reverse=True)[:25]:
    print(f"  {g[0]:.3f}  {g[1]}  ->  {g[2]}")
