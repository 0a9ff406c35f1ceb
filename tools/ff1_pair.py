"""One FF1-shape GEMM (M=8192, N=49152, K=12288, NN, bf16) by tess and by
cuBLAS, for side-by-side ncu counter captures."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2105_14500_b200 as tess  # noqa: E402

M, N, K = [int(v) for v in os.environ.get("MNK", "8192,49152,12288").split(",")]
dev = torch.device("cuda", 0)
ctx = tess.init_local(tess.GridSpec(1, 1))[0]
a = torch.randn(M, K, device=dev, dtype=torch.bfloat16)
b = torch.randn(K, N, device=dev, dtype=torch.bfloat16)
c = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
st = torch.cuda.current_stream().cuda_stream
for _ in range(2):
    ctx.matmul("nn", "bf16", a.data_ptr(), M, K, b.data_ptr(), K, N, c.data_ptr(), c_dtype="bf16",
               stream=st)
    torch.matmul(a, b, out=c)
torch.cuda.synchronize()
ctx.close()
print("ok")
