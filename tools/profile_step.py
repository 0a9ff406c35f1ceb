"""One cfg4 block fwd+bwd at [1,1,1] with per-launch GEMM timing grouped by
(kernel, shape, epilogue) -- where the step's GEMM time goes."""
import json
import os
import sys

os.environ["TESS_PROFILE_DETAIL"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

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


for _ in range(2):
    step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
step()
e1.record()
torch.cuda.synchronize()
step_ms = e0.elapsed_time(e1)
tess.profile_enable(True)
step()
torch.cuda.synchronize()
k = tess.profile_kernels()
tess.profile_enable(False)
tot = sum(v[0] for v in k.values())
print(json.dumps({"step_ms": step_ms, "gemm_ms": tot}))
for name, (ms, fl, n, by) in sorted(k.items(), key=lambda kv: -kv[1][0]):
    rate = f"{fl / ms / 1e9:7.1f} TF/s" if fl else f"{by / ms / 1e6:7.1f} GB/s"
    print(f"{ms:8.3f} ms {100 * ms / step_ms:5.1f}%  {rate}  x{int(n):3d}  {name}")
ctx.close()
