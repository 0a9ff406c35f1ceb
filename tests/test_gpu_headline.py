"""Parity pinned at the configurations the benchmark numbers come from.

The bench's tensor launches are mostly the 256 x 512 pair-tile kernel
(`gemm_bf16_2cta_kernel<*,*,512>`, NH = 2) with the TMA-store epilogues
(Store, Accum = TMA reduce-add, Resid, Gelu = z and h stores, DGelu). The
dispatcher picks that tile only when it does not cost a wave, so small test
shapes land elsewhere. This file checks those exact kernels:

  * `test_nh2_forced_suite` re-runs the bf16 oracle suites in a child
    process with TESS_GEMM_NH=2 (every GEMM with N > 256 on the 512-wide
    tile), plus `test_nh2_block_vs_oracle_*` (child only): a bf16 block
    fwd+bwd at b=4 s=128 h=1024 on [1,1,1], [1,1,2], [2,2,1], [2,2,2] against
    the fp64 oracle (reference layers.cpp:460-487), asserting through the
    detailed GEMM profile that the 512-tile kernel ran with the Store, Accum,
    Resid, Gelu and DGelu epilogues;
  * `test_cfg4_block_vs_torch`: the benchmark's own layer (cfg4: h=12288,
    96 heads, s=2048; b=1) on [1,1,1] with the dispatcher's natural tile
    choice, against a PyTorch fp32 autograd block on the same bf16 inputs;
  * `test_cfg2_linear_vs_torch`: BASELINE config 2's Linear
    (X 16384x4096, W 4096x16384: NN forward, NT dgrad, TN wgrad) against
    torch fp32 products of the same bf16 inputs.

Tolerances (relative Frobenius, stated per SURVEY App. C): whole bf16
layer <= 2e-2; a single GEMM with fp32 output <= 1e-4 (identical bf16
inputs, fp32 accumulation in both), with bf16 output <= 5e-3.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = os.environ.get("TESS_GEMM_NH") == "2"

EPI = {"store": 0, "accum": 1, "resid": 2, "gelu": 3, "dgelu": 4}


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


def wide_tile_epilogues(kernels):
    """Epilogue ids that ran on the 256 x 512 pair-tile kernel (detailed
    profile keys: '<kernel> M=.. N=.. K=.. b=.. epi=<n>')."""
    out = set()
    for k in kernels:
        name = k.split(" ")[0]
        if name.startswith("gemm_bf16_2cta_kernel<") and name.endswith(",512>"):
            out.add(int(k.rsplit("epi=", 1)[1]))
    return out


# ------------------------------------------------ child: NH = 2 forced
NH2_SHAPE = (4, 128, 1024, 8)  # b, s, h, heads: T = 512, h/q >= 512 on q = 2
_oracle_cache = {}


def _nh2_inputs(orc):
    if "in" not in _oracle_cache:
        b, s, h, nh = NH2_SHAPE
        x = bf16r(orc.random_matrix(b * s, h, 31, 0))
        dy = bf16r(orc.random_matrix(b * s, h, 31, 2))
        P = orc.random_block_params(h, 31, 100)
        P = {k: (bf16r(v) if k.startswith("w_") else v.astype(np.float32).astype(np.float64))
             for k, v in P.items()}
        _oracle_cache["in"] = (x, dy, P, orc.layer_run("block", x, dy, P, b, s, nh))
    return _oracle_cache["in"]


@pytest.mark.skipif(not CHILD, reason="runs in the TESS_GEMM_NH=2 child (test_nh2_forced_suite)")
@pytest.mark.parametrize("q,d,allow", [(1, 1, False), (1, 2, True), (2, 1, False),
                                       (2, 2, False)])
def test_nh2_block_vs_oracle(tess, orc, q, d, allow):
    b, s, h, nh = NH2_SHAPE
    x, dy, P, want = _nh2_inputs(orc)
    tess.profile_enable(True, detail=True)
    try:
        res = tess.layer_run("block", x, dy, P, tess.LayerDims(b, s, h, nh),
                             tess.GridSpec(q, d, allow), dtype="bf16")
        kernels = tess.profile_kernels()
    finally:
        tess.profile_enable(False)
    errs = {"y": frob(res.y, want["y"]), "dx": frob(res.dx, want["dx"])}
    for k, v in want["grads"].items():
        errs[k] = frob(res.grads[k], v)
    print(f"nh2 block [{q},{q},{d}] errs {errs}")
    assert max(errs.values()) <= 2e-2, errs
    rows = b * s // (d * q)
    if rows > 128:  # the pair kernel needs M > 128 (rows per rank)
        ran = wide_tile_epilogues(kernels)
        need = {EPI["store"], EPI["gelu"], EPI["resid"]}
        if q == 1:  # q > 1: dh is row-reduced first, GeLU' is applied after the reduce
            need.add(EPI["dgelu"])
        assert need <= ran, (sorted(ran), sorted(kernels))


@pytest.mark.skipif(not CHILD, reason="runs in the TESS_GEMM_NH=2 child (test_nh2_forced_suite)")
def test_nh2_accumulate_epilogue_vs_oracle(tess, orc):
    """Weight-gradient accumulation (accumulate=True: the TN epilogue becomes a
    TMA reduce-add into the fp32 gradient) on the 512-wide tile: two
    backward passes into the same gradients give twice the oracle's."""
    import torch
    b, s, h, nh = NH2_SHAPE
    x, dy, P, want = _nh2_inputs(orc)
    dev = torch.device("cuda", 0)
    bf = torch.bfloat16
    names = ("w_qkv", "w_proj", "w_ff1", "w_ff2")
    W = [torch.tensor(P[k], dtype=torch.float32, device=dev).to(bf).contiguous() for k in names]
    LN = [torch.tensor(P[k], dtype=torch.float32, device=dev).reshape(-1).contiguous()
          for k in ("ln1_gain", "ln1_bias", "ln2_gain", "ln2_bias")]
    xt = torch.tensor(x, dtype=torch.float32, device=dev).to(bf)
    dyt = torch.tensor(dy, dtype=torch.float32, device=dev).to(bf)
    shard = tess.BlockShardC(*[t.data_ptr() for t in W + LN], 1e-5)
    dims = tess.LayerDims(b, s, h, nh)
    G = [torch.zeros(t.shape, device=dev) for t in W + LN]
    grads = tess.BlockGradsC(*[t.data_ptr() for t in G])
    ctx = tess.init_local(tess.GridSpec(1, 1))[0]
    st = torch.cuda.current_stream().cuda_stream
    tess.profile_enable(True, detail=True)
    try:
        y, dx = torch.empty_like(xt), torch.empty_like(xt)
        for _ in range(2):
            ctx.layer_forward("block", "bf16", dims, shard, xt.data_ptr(), y.data_ptr(), stream=st)
            ctx.layer_backward("block", "bf16", dims, shard, dyt.data_ptr(), dx.data_ptr(), grads,
                               accumulate=True, stream=st)
        torch.cuda.synchronize()
        kernels = tess.profile_kernels()
    finally:
        tess.profile_enable(False)
        ctx.close()
    assert EPI["accum"] in wide_tile_epilogues(kernels), sorted(kernels)
    for k, g in zip(tess.PARAM_NAMES, G):
        ref = 2 * want["grads"][k].reshape(g.shape)
        assert frob(g.double().cpu().numpy(), ref) <= 2e-2, k


def test_nh2_forced_suite(tess):
    """The bf16 oracle suites re-run with every N > 256 GEMM on the 256 x 512
    pair tile (TESS_GEMM_NH=2 is read once per process, hence the child)."""
    if CHILD:
        pytest.skip("already the child")
    env = dict(os.environ, TESS_GEMM_NH="2")
    cmd = [sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
           "tests/test_gpu_headline.py::test_nh2_block_vs_oracle",
           "tests/test_gpu_headline.py::test_nh2_accumulate_epilogue_vs_oracle",
           "tests/test_gpu_parity.py::test_layers_bf16",
           "tests/test_gpu_parity.py::test_train_toy_bf16",
           "tests/test_gpu_parity.py::test_block_fused_layernorm_bf16",
           "tests/test_gpu_attention.py::test_fused_attention_vs_oracle"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=1800)
    tail = (r.stdout + r.stderr)[-4000:]
    assert r.returncode == 0, tail
    assert " passed" in r.stdout and "skipped" not in r.stdout.split("\n")[-2], tail


# ------------------------------------------- cfg4 block vs torch fp32
def torch_block(x, P, dy, b, s, nh, eps=1e-5):
    """fp32 autograd restatement of the reference block (layers.cpp:460-487):
    r1 = x + attn(LN1 x), y = r1 + ff(LN2 r1); attention with per-head
    interleaved (Q|K|V) columns and no mask (layers.cpp:383-414); exact erf
    GeLU (layers.cpp:25-42); LayerNorm with population variance."""
    import torch
    F = torch.nn.functional
    x = x.clone().requires_grad_(True)
    P = {k: v.clone().requires_grad_(True) for k, v in P.items()}
    h = x.shape[1]
    hd = h // nh
    a = F.layer_norm(x, (h,), P["ln1_gain"], P["ln1_bias"], eps)
    qkv = (a @ P["w_qkv"]).view(b, s, nh, 3, hd)
    qh, kh, vh = (qkv[:, :, :, i].permute(0, 2, 1, 3) for i in range(3))
    p = torch.softmax(qh @ kh.transpose(-1, -2) / hd ** 0.5, dim=-1)
    o = (p @ vh).permute(0, 2, 1, 3).reshape(b * s, h)
    r1 = x + o @ P["w_proj"]
    c = F.layer_norm(r1, (h,), P["ln2_gain"], P["ln2_bias"], eps)
    y = r1 + F.gelu(c @ P["w_ff1"]) @ P["w_ff2"]
    y.backward(dy)
    return y.detach(), x.grad, {k: v.grad for k, v in P.items()}


def test_cfg4_block_vs_torch(tess):
    """BASELINE cfg4's layer at its real shape (h=12288, 96 heads, s=2048;
    b=1 sample), [1,1,1], dispatcher's own tile choice = the bench's kernels."""
    import torch
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    torch.manual_seed(4)
    b, s, h, nh = 1, 2048, 12288, 96
    dev = torch.device("cuda", 0)
    bf = torch.bfloat16

    def u(shape, scale=1.0):
        return ((torch.rand(shape, device=dev) * 2 - 1) * scale).to(bf).float()
    ws = h ** -0.5
    P = {"w_qkv": u((h, 3 * h), ws), "w_proj": u((h, h), ws), "w_ff1": u((h, 4 * h), ws),
         "w_ff2": u((4 * h, h), ws),
         "ln1_gain": 1 + (torch.rand(h, device=dev) * 2 - 1) * 0.1,
         "ln1_bias": (torch.rand(h, device=dev) * 2 - 1) * 0.1,
         "ln2_gain": 1 + (torch.rand(h, device=dev) * 2 - 1) * 0.1,
         "ln2_bias": (torch.rand(h, device=dev) * 2 - 1) * 0.1}
    x = u((b * s, h))
    dy = u((b * s, h))

    # device path first (frees its buffers before the fp32 reference runs)
    names = tess.PARAM_NAMES
    W = [P[k].to(bf).contiguous() for k in names[:4]]
    LN = [P[k].contiguous() for k in names[4:]]
    G = [torch.zeros(t.shape, device=dev) for t in W + LN]
    xb, dyb = x.to(bf), dy.to(bf)
    y, dx = torch.empty_like(xb), torch.empty_like(xb)
    shard = tess.BlockShardC(*[t.data_ptr() for t in W + LN], 1e-5)
    grads = tess.BlockGradsC(*[t.data_ptr() for t in G])
    dims = tess.LayerDims(b, s, h, nh)
    ctx = tess.init_local(tess.GridSpec(1, 1))[0]
    st = torch.cuda.current_stream().cuda_stream
    tess.profile_enable(True, detail=True)
    try:
        ctx.layer_forward("block", "bf16", dims, shard, xb.data_ptr(), y.data_ptr(), stream=st)
        ctx.layer_backward("block", "bf16", dims, shard, dyb.data_ptr(), dx.data_ptr(), grads,
                           stream=st)
        torch.cuda.synchronize()
        kernels = tess.profile_kernels()
    finally:
        tess.profile_enable(False)
        ctx.close()
    del W, xb, dyb
    ran = wide_tile_epilogues(kernels)
    assert {EPI["store"], EPI["gelu"], EPI["resid"], EPI["dgelu"]} <= ran, sorted(kernels)
    assert any(k.startswith("attn_fwd_kernel<128>") for k in kernels)
    assert any(k.startswith("attn_bwd_kv_kernel<128>") for k in kernels)
    assert any(k.startswith("attn_dq_kernel<128>") for k in kernels)

    ry, rdx, rg = torch_block(x, P, dy, b, s, nh)

    def rel(a, r):
        return ((a.float() - r).norm() / r.norm()).item()
    errs = {"y": rel(y, ry), "dx": rel(dx, rdx)}
    for k, g in zip(names, G):
        errs[k] = rel(g.reshape(rg[k].shape), rg[k])
    print(f"cfg4 block errs {errs}")
    assert max(errs.values()) <= 2e-2, errs


# -------------------------------------------- cfg2 Linear vs torch fp32
@pytest.mark.parametrize("variant", ["nn", "nt", "tn"])
def test_cfg2_linear_vs_torch(tess, variant):
    """Config 2 (X 16384x4096, W 4096x16384, dY 16384x16384, bf16): the three
    Tesseract products of a Linear fwd+bwd (layers.cpp:349-379 pattern;
    algorithms.cpp:34-76 at [1,1,1]) with the output types the layers use:
    NN y (bf16), NT dX (bf16), TN dW (fp32)."""
    import torch
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.manual_seed(2)
    dev = torch.device("cuda", 0)
    bf = torch.bfloat16
    T, K, N = 16384, 4096, 16384
    if variant == "nn":
        a = torch.randn(T, K, device=dev, dtype=bf)
        b = (torch.randn(K, N, device=dev) * K ** -0.5).to(bf)
        ref, dims, out = a.float() @ b.float(), (T, K, K, N), ("bf16", (T, N))
    elif variant == "nt":
        a = torch.randn(T, N, device=dev, dtype=bf)
        b = (torch.randn(K, N, device=dev) * K ** -0.5).to(bf)
        ref, dims, out = a.float() @ b.float().t(), (T, N, K, N), ("bf16", (T, K))
    else:
        a = torch.randn(T, K, device=dev, dtype=bf)
        b = torch.randn(T, N, device=dev, dtype=bf)
        ref, dims, out = a.float().t() @ b.float(), (T, K, T, N), ("f32", (K, N))
    c = torch.zeros(out[1], device=dev, dtype=bf if out[0] == "bf16" else torch.float32)
    ctx = tess.init_local(tess.GridSpec(1, 1))[0]
    tess.profile_enable(True, detail=True)
    try:
        ctx.matmul(variant, "bf16", a.data_ptr(), dims[0], dims[1], b.data_ptr(), dims[2], dims[3],
                   c.data_ptr(), c_dtype=out[0], stream=torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        kernels = tess.profile_kernels()
    finally:
        tess.profile_enable(False)
        ctx.close()
    assert EPI["store"] in wide_tile_epilogues(kernels), sorted(kernels)
    err = ((c.float() - ref).norm() / ref.norm()).item()
    print(f"cfg2 {variant} err {err:.3e}")
    assert err <= (5e-3 if out[0] == "bf16" else 1e-4), err
