"""One FF1-shape GEMM (8192 x 49152 x 12288, bf16 -> bf16) by cuBLAS
(torch.matmul) and by the tess tcgen05 kernel, for an ncu metrics pass that
compares per-flop data movement and instruction counts of the two (where the
energy of a power-capped GEMM goes besides the MMAs). MODE=1 only tess,
MODE=2 only cuBLAS, default both."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2105_14500_b200 as tess  # noqa: E402

M, N, K = 8192, 49152, 12288
dev = torch.device("cuda", 0)
a = torch.randn(M, K, device=dev, dtype=torch.bfloat16)
b = torch.randn(K, N, device=dev, dtype=torch.bfloat16)
c = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
mode = int(os.environ.get("MODE", "0"))
ctx = tess.init_local(tess.GridSpec(1, 1))[0]
st = torch.cuda.current_stream().cuda_stream
for _ in range(2):
    if mode in (0, 2):
        torch.matmul(a, b, out=c)
    if mode in (0, 1):
        ctx.matmul("nn", "bf16", a.data_ptr(), M, K, b.data_ptr(), K, N, c.data_ptr(),
                   c_dtype="bf16", stream=st)
torch.cuda.synchronize()
ctx.close()
