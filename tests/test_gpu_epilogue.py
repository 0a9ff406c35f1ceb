"""Fused bias / GeLU / dropout-scale / residual epilogue of the tcgen05 GEMM
(tess_matmul_ex; north_star: "bias/GeLU/dropout-scale fused in the
epilogue"). The reference's blocks have no linear biases or dropout
(layers.hpp:42-49), so the check is against a torch fp32 restatement of the
same formula on the same bf16 inputs, with the mask from the host
restatement of the counter hash (tess_dropout_keep):

    v = A B + bias ; [GeLU: z = v, v = gelu(v)] ; v = keep ? v/(1-p) : 0 ;
    [v += residual] ; [C += v with accumulate]

Shapes reach the 1-CTA kernel (N <= 256) and the 256x512 pair tile with the
TMA-store epilogue (TESS_GEMM_NH defaults: N >= 512 shapes). Tolerances:
bf16 output relative Frobenius <= 5e-3, fp32 output <= 1e-4; dropped
elements are exactly zero. The sharded case ([2,2,1], one thread per rank)
drops exactly the unsharded product's elements (the mask is a function of
the global coordinate).
"""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tess():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2105_14500_b200 as t
    return t


def frob(v, r):
    return float(np.linalg.norm(v - r) / max(np.linalg.norm(r), 1e-30))


def _inputs(M, K, N, seed):
    import torch
    g = torch.Generator().manual_seed(seed)
    a = (torch.rand(M, K, generator=g) * 2 - 1).to(torch.bfloat16)
    b = ((torch.rand(K, N, generator=g) * 2 - 1) / K ** 0.5).to(torch.bfloat16)
    bias = torch.rand(N, generator=g) * 0.4 - 0.2
    res = (torch.rand(M, N, generator=g) * 2 - 1).to(torch.bfloat16)
    return a, b, bias, res


def _reference(tess, a, b, bias, res, mode, p, seed, row0=0, col0=0, c0=None):
    import torch
    v = a.float() @ b.float() + bias
    z = v.clone()
    if mode == "gelu":
        v = torch.nn.functional.gelu(v)
    if p > 0:
        rr, cc = np.meshgrid(np.arange(a.shape[0]) + row0, np.arange(b.shape[1]) + col0,
                             indexing="ij")
        keep = torch.from_numpy(tess.dropout_keep(seed, rr, cc, p))
        v = torch.where(keep, v / (1 - p), torch.zeros_like(v))
    else:
        keep = None
    if mode == "resid":
        v = v + res.float()
    if mode == "accum":
        v = v + c0
    return v, z, keep


@pytest.mark.parametrize("M,K,N", [(512, 256, 192), (1024, 512, 1024), (640, 384, 2048)])
@pytest.mark.parametrize("mode,p", [("store", 0.1), ("gelu", 0.2), ("resid", 0.3),
                                    ("accum", 0.1), ("store", 0.0), ("gelu", 0.0)])
def test_fused_epilogue_local(tess, M, K, N, mode, p):
    import torch
    ctx = tess.init_local(tess.GridSpec(1, 1))[0]
    try:
        seed = 0x5EED + M + N
        a, b, bias, res = _inputs(M, K, N, M * 7 + N)
        da, db, dbias, dres = a.cuda(), b.cuda(), bias.cuda(), res.cuda()
        out_t = torch.float32 if mode == "accum" else torch.bfloat16
        c0 = torch.rand(M, N) if mode == "accum" else None
        dc = c0.cuda() if c0 is not None else torch.empty(M, N, dtype=out_t, device="cuda")
        dz = torch.empty(M, N, dtype=out_t, device="cuda")
        ep = {"bias": dbias.data_ptr(), "gelu": int(mode == "gelu"),
              "pre_activation": dz.data_ptr() if mode == "gelu" else None, "dropout_p": p,
              "dropout_seed": seed, "row0": 0, "col0": 0,
              "residual": dres.data_ptr() if mode == "resid" else None}
        ctx.matmul("nn", "bf16", da.data_ptr(), M, K, db.data_ptr(), K, N, dc.data_ptr(),
                   c_dtype="f32" if mode == "accum" else "bf16", accumulate=mode == "accum",
                   epilogue=ep)
        torch.cuda.synchronize()
        want, z, keep = _reference(tess, a, b, bias, res, mode, p, seed, c0=c0)
        got = dc.float().cpu()
        tol = 1e-4 if mode == "accum" else 5e-3
        assert frob(got.numpy(), want.numpy()) <= tol
        if mode == "gelu":
            assert frob(dz.float().cpu().numpy(), z.numpy()) <= 5e-3
        if keep is not None and mode in ("store", "gelu"):
            assert bool((got[~keep] == 0).all())
    finally:
        ctx.close()


def test_fused_epilogue_sharded_mask(tess):
    """NN on [2,2,1] with bias + dropout: every block equals the unsharded
    reference's block (mask from the global coordinate)."""
    import torch
    q, d = 2, 1
    grid = tess.GridSpec(q, d)
    M, K, N, p, seed = 1024, 512, 1024, 0.25, 4242
    a, b, bias, res = _inputs(M, K, N, 99)
    want, _, keep = _reference(tess, a, b, bias, res, "store", p, seed)
    ctxs = tess.init_local(grid)
    rb, kb, nb = M // (q * d), K // q, N // q
    outs, errs = {}, []

    def run(r):
        try:
            cx = ctxs[r]
            c = grid.coord_of(r)
            h = c.i + c.k * q  # block row of TesseractA (grid.cpp:63-69)
            la = a[h * rb:(h + 1) * rb, c.j * kb:(c.j + 1) * kb].contiguous().cuda()
            lb = b[c.i * kb:(c.i + 1) * kb, c.j * nb:(c.j + 1) * nb].contiguous().cuda()
            lbias = bias[c.j * nb:(c.j + 1) * nb].contiguous().cuda()
            lc = torch.empty(rb, nb, dtype=torch.bfloat16, device="cuda")
            cx.matmul("nn", "bf16", la.data_ptr(), rb, kb, lb.data_ptr(), kb, nb, lc.data_ptr(),
                      c_dtype="bf16",
                      epilogue={"bias": lbias.data_ptr(), "gelu": 0, "pre_activation": None,
                                "dropout_p": p, "dropout_seed": seed, "row0": h * rb,
                                "col0": c.j * nb, "residual": None})
            torch.cuda.synchronize()
            outs[r] = (h, c.j, lc.float().cpu())
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=run, args=(r,)) for r in range(grid.size())]
    [t.start() for t in th]
    [t.join() for t in th]
    for cx in ctxs:
        cx.close()
    assert not errs, errs
    for h, j, blk in outs.values():
        w = want[h * rb:(h + 1) * rb, j * nb:(j + 1) * nb]
        kp = keep[h * rb:(h + 1) * rb, j * nb:(j + 1) * nb]
        assert frob(blk.numpy(), w.numpy()) <= 5e-3
        assert bool((blk[~kp] == 0).all())


def test_fused_epilogue_rejections(tess):
    import torch
    ctx = tess.init_local(tess.GridSpec(1, 1))[0]
    try:
        a = torch.zeros(128, 128, dtype=torch.float32, device="cuda")
        with pytest.raises(tess.UnsupportedError):
            ctx.matmul("nn", "f32", a.data_ptr(), 128, 128, a.data_ptr(), 128, 128, a.data_ptr(),
                       epilogue={"bias": a.data_ptr(), "gelu": 0, "pre_activation": None,
                                 "dropout_p": 0.0, "dropout_seed": 0, "row0": 0, "col0": 0,
                                 "residual": None})
    finally:
        ctx.close()
