"""The optional 4-CTA multicast GEMM (TESS_GEMM_MC=1, kernels/gemm_sm100.cu
MC = 2 plus its pair companion) against the default pair kernel on the same
inputs: both are fp32-accumulated bf16 products, equal up to summation order
(the serpentine K direction depends on the launch's wave width). Run in a
subprocess because the switch is read once per process."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = r"""
import sys
import numpy as np
import torch
sys.path.insert(0, sys.argv[1])
import paper_2105_14500_b200 as tess
dev = torch.device("cuda", 0)
ctx = tess.init_local(tess.GridSpec(1, 1))[0]
st = torch.cuda.current_stream().cuda_stream
out = {}
g = torch.Generator(device=dev).manual_seed(3)
# shapes that take the 256 x 512 pair tiles (where the multicast variant applies)
for name, (M, K, N, v) in {"nn": (8192, 1024, 12288, "nn"), "nt": (8192, 1024, 12288, "nt"),
                           "tn": (8192, 1024, 12288, "tn")}.items():
    sa = (M, K) if v != "tn" else (K, M)
    sb = {"nn": (K, N), "nt": (N, K), "tn": (K, N)}[v]
    a = torch.randn(sa, device=dev, generator=g).to(torch.bfloat16)
    b = (torch.randn(sb, device=dev, generator=g) * K ** -0.5).to(torch.bfloat16)
    c = torch.zeros(M, N, device=dev, dtype=torch.float32)
    ctx.matmul(v, "bf16", a.data_ptr(), *sa, b.data_ptr(), *sb, c.data_ptr(), stream=st)
    torch.cuda.synchronize()
    out[name] = c.cpu().numpy()
ctx.close()
np.savez(sys.argv[2], **out)
"""


def _run(tmp_path, mc):
    path = str(tmp_path / f"mc{mc}.npz")
    env = dict(os.environ, TESS_GEMM_MC=str(mc), TESS_GEMM_MC_DEBUG="1")
    r = subprocess.run([sys.executable, "-c", WORKER, ROOT, path], check=True, env=env,
                       timeout=600, capture_output=True, text=True)
    # the multicast launcher reports its cluster count once per instantiation
    assert ("active clusters" in r.stderr) == (mc == 1), r.stderr[-2000:]
    return np.load(path)


def test_multicast_gemm_matches_pair_kernel(tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    base, mc = _run(tmp_path, 0), _run(tmp_path, 1)
    for k in base.files:
        rel = np.linalg.norm(mc[k] - base[k]) / np.linalg.norm(base[k])
        assert rel <= 1e-5, (k, rel)
