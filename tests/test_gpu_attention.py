"""Fused tcgen05 attention (kernels/attention_sm100.cu) parity.

The bf16 attention layer runs the fused forward / backward kernels whenever
head_dim is 64 or 128 and seq % 8 == 0. They are checked
  * against the fp64 oracle (reference layers.cpp:383-456 restated) through
    tess.layer_run on several grids, ragged sequence lengths included, at the
    bf16-layer tolerance of test_gpu_parity.py (relative Frobenius <= 2e-2);
  * at the full cfg4 head shape (s = 2048, hd = 128) against a plain PyTorch
    fp32 attention layer on the same bf16 inputs (relative Frobenius <= 2e-2);
  * for bitwise run-to-run determinism (no atomics anywhere in the path).
"""
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


def bf16r(a):
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def frob(v, r):
    return np.linalg.norm(v - r) / max(np.linalg.norm(r), 1e-30)


def _inputs(orc, b, s, h, seed):
    x = bf16r(orc.random_matrix(b * s, h, seed, 0))
    dy = bf16r(orc.random_matrix(b * s, h, seed, 2))
    P = orc.random_block_params(h, seed, 100)
    P = {k: (bf16r(v) if k.startswith("w_") else v.astype(np.float32).astype(np.float64))
         for k, v in P.items()}
    return x, dy, P


# (batch, seq, hidden, heads, q, d, allow): head_dim 128 and 64, ragged seq
# (200, 136: neither a multiple of the 64-query nor the 128-key tile), grids
# with several local heads and samples.
SHAPES = [
    (2, 256, 256, 2, 1, 1, False),
    (2, 200, 128, 2, 1, 1, False),
    (4, 128, 512, 4, 2, 2, False),
    (4, 136, 256, 4, 2, 1, False),
    (2, 384, 256, 2, 1, 2, True),
]


@pytest.mark.parametrize("b,s,h,nh,q,d,allow", SHAPES)
@pytest.mark.parametrize("op", ["attention", "block"])
def test_fused_attention_vs_oracle(tess, orc, b, s, h, nh, q, d, allow, op):
    x, dy, P = _inputs(orc, b, s, h, 21)
    want = orc.layer_run(op, x, dy, P, b, s, nh)
    tess.profile_enable(True)
    try:
        res = tess.layer_run(op, x, dy, P, tess.LayerDims(b, s, h, nh),
                             tess.GridSpec(q, d, allow), dtype="bf16")
        kernels = tess.profile_kernels()
    finally:
        tess.profile_enable(False)
    hd = h // nh
    assert f"attn_fwd_kernel<{hd}>" in kernels, kernels
    assert f"attn_bwd_kv_kernel<{hd}>" in kernels and f"attn_dq_kernel<{hd}>" in kernels, kernels
    errs = {"y": frob(res.y, want["y"]), "dx": frob(res.dx, want["dx"])}
    for k, v in want["grads"].items():
        if np.abs(v).max() > 0:
            errs[k] = frob(res.grads[k], v)
    assert max(errs.values()) <= 2e-2, errs


def _torch_attention_layer(x, wqkv, wproj, dy, b, s, nh):
    """fp32 autograd reference of the attention op (reference layers.cpp:383-456):
    qkv = x Wqkv with per-head interleaved (Q|K|V) columns, no mask."""
    import torch
    x = x.clone().requires_grad_(True)
    wqkv = wqkv.clone().requires_grad_(True)
    wproj = wproj.clone().requires_grad_(True)
    h = x.shape[1]
    hd = h // nh
    qkv = (x @ wqkv).view(b, s, nh, 3, hd)
    qh, kh, vh = (qkv[:, :, :, i].permute(0, 2, 1, 3) for i in range(3))
    p = torch.softmax(qh @ kh.transpose(-1, -2) / hd ** 0.5, dim=-1)
    o = (p @ vh).permute(0, 2, 1, 3).reshape(b * s, h)
    y = o @ wproj
    y.backward(dy)
    return y.detach(), x.grad, wqkv.grad, wproj.grad


def _run_attention_device(tess, b, s, h, nh, x, wqkv, wproj, dy):
    import torch
    dev = x.device
    ctx = tess.init_local(tess.GridSpec(1, 1))[0]
    try:
        bf = torch.bfloat16
        W = [wqkv.to(bf).contiguous(), wproj.to(bf).contiguous(),
             torch.zeros(8, device=dev, dtype=bf), torch.zeros(8, device=dev, dtype=bf)]
        LN = [torch.ones(h, device=dev), torch.zeros(h, device=dev),
              torch.ones(h, device=dev), torch.zeros(h, device=dev)]
        xb, dyb = x.to(bf).contiguous(), dy.to(bf).contiguous()
        y, dx = torch.empty_like(xb), torch.empty_like(xb)
        G = [torch.zeros(wqkv.shape, device=dev), torch.zeros(wproj.shape, device=dev),
             torch.zeros(8, device=dev), torch.zeros(8, device=dev)] + \
            [torch.zeros(h, device=dev) for _ in range(4)]
        shard = tess.BlockShardC(*[t.data_ptr() for t in W + LN], 1e-5)
        grads = tess.BlockGradsC(*[t.data_ptr() for t in G])
        dims = tess.LayerDims(b, s, h, nh)
        st = torch.cuda.current_stream().cuda_stream
        ctx.layer_forward("attention", "bf16", dims, shard, xb.data_ptr(), y.data_ptr(), stream=st)
        ctx.layer_backward("attention", "bf16", dims, shard, dyb.data_ptr(), dx.data_ptr(), grads,
                           stream=st)
        torch.cuda.synchronize()
        return y.float(), dx.float(), G[0], G[1]
    finally:
        ctx.close()


def _rel(a, b):
    import torch
    return (torch.linalg.norm(a - b) / torch.linalg.norm(b)).item()


def test_fused_attention_cfg4_head_shape_vs_torch(tess):
    """s = 2048, hd = 128 (BASELINE cfg4 per-head shape), 4 heads, 1 sample."""
    import torch
    torch.manual_seed(0)
    b, s, nh, hd = 1, 2048, 4, 128
    h = nh * hd
    dev = torch.device("cuda", 0)

    def bf(t):
        return t.to(torch.bfloat16).float()
    x = bf(torch.randn(b * s, h, device=dev))
    wqkv = bf(torch.randn(h, 3 * h, device=dev) * h ** -0.5)
    wproj = bf(torch.randn(h, h, device=dev) * h ** -0.5)
    dy = bf(torch.randn(b * s, h, device=dev))
    ry, rdx, rgq, rgp = _torch_attention_layer(x, wqkv, wproj, dy, b, s, nh)
    gy, gdx, ggq, ggp = _run_attention_device(tess, b, s, h, nh, x, wqkv, wproj, dy)
    errs = {"y": _rel(gy, ry), "dx": _rel(gdx, rdx), "w_qkv": _rel(ggq, rgq),
            "w_proj": _rel(ggp, rgp)}
    assert max(errs.values()) <= 2e-2, errs


@pytest.mark.parametrize("b,s,nh,hd", [(4, 392, 40, 64), (3, 520, 24, 128)])
def test_fused_attention_persistent_units_vs_torch(tess, b, s, nh, hd):
    """More (sample, head, tile) units than SMs, so every persistent CTA of
    the two backward passes runs several units back to back (ring phases,
    K/V and Q/dO reloads, accumulator hand-over across units), with ragged
    sequences (392 = 3 x 128 + 8, 520 = 4 x 128 + 8) and both head dims."""
    import torch
    torch.manual_seed(1)
    h = nh * hd
    dev = torch.device("cuda", 0)

    def bf(t):
        return t.to(torch.bfloat16).float()
    x = bf(torch.randn(b * s, h, device=dev))
    wqkv = bf(torch.randn(h, 3 * h, device=dev) * h ** -0.5)
    wproj = bf(torch.randn(h, h, device=dev) * h ** -0.5)
    dy = bf(torch.randn(b * s, h, device=dev))
    ry, rdx, rgq, rgp = _torch_attention_layer(x, wqkv, wproj, dy, b, s, nh)
    gy, gdx, ggq, ggp = _run_attention_device(tess, b, s, h, nh, x, wqkv, wproj, dy)
    errs = {"y": _rel(gy, ry), "dx": _rel(gdx, rdx), "w_qkv": _rel(ggq, rgq),
            "w_proj": _rel(ggp, rgp)}
    assert max(errs.values()) <= 2e-2, errs


def test_fused_attention_deterministic(tess, orc):
    b, s, h, nh = 2, 256, 256, 2
    x, dy, P = _inputs(orc, b, s, h, 5)
    runs = [tess.layer_run("attention", x, dy, P, tess.LayerDims(b, s, h, nh),
                           tess.GridSpec(1, 1), dtype="bf16") for _ in range(2)]
    assert (runs[0].y == runs[1].y).all() and (runs[0].dx == runs[1].dx).all()
    for k in runs[0].grads:
        assert (runs[0].grads[k] == runs[1].grads[k]).all(), k
