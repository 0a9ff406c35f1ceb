"""Numerics + identity check of the GEMM on the cfg4 FF1 / FF2 shapes against
torch.matmul (fp32 accumulate on both sides): prints the relative Frobenius
error and the kernel names launched (tess.profile_kernels)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2105_14500_b200 as tess  # noqa: E402

dev = torch.device("cuda", 0)
ctx = tess.init_local(tess.GridSpec(1, 1))[0]
st = torch.cuda.current_stream().cuda_stream
torch.manual_seed(0)
for (M, K, N) in [(8192, 12288, 49152), (8192, 49152, 12288), (8192, 12288, 12288)]:
    a = torch.randn(M, K, device=dev, dtype=torch.bfloat16)
    b = torch.randn(K, N, device=dev, dtype=torch.bfloat16) * K ** -0.5
    c = torch.empty(M, N, device=dev, dtype=torch.float32)
    tess.profile_enable(True)
    ctx.matmul("nn", "bf16", a.data_ptr(), M, K, b.data_ptr(), K, N, c.data_ptr(), stream=st)
    torch.cuda.synchronize()
    names = tess.profile_kernels()
    tess.profile_enable(False)
    ref = (a.float() @ b.float())
    err = (torch.linalg.norm(c - ref) / torch.linalg.norm(ref)).item()
    print(M, K, N, "rel_frob", f"{err:.3e}", list(names)[:2], flush=True)
    assert err < 1e-4, err
ctx.close()
