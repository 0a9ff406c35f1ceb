"""One cfg4 block fwd+bwd at [1,1,1] bracketed by cudaProfilerStart/Stop, for
`ncu --profile-from-start off` launch lists (per-kernel share of one step):

  ncu --profile-from-start off --metrics gpu__time_duration.sum \
      --clock-control none --csv --log-file gpurun_out/launches.csv \
      python tools/ncu_step.py
"""
import os
import sys

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


step()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
step()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("ok")
