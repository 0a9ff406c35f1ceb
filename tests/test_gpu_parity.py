"""GPU parity: the CUDA path (through the C-ABI) against the fp64 oracle.

Tolerances (north star + SURVEY App. C):
  * partition / gather: bit-exact;
  * fp32 mode: rel_diff (max|diff| / max|ref|, matrix.cpp:138-140) <= 1e-5
    against the oracle run on the same fp32-rounded inputs;
  * bf16 mode (tcgen05, fp32 accumulate, fp32 output before any cast):
    relative Frobenius <= 1e-4 vs the oracle on identical bf16-rounded
    inputs, <= 5e-3 vs the oracle on the original fp64 inputs;
  * bf16 layers (intermediates stored in bf16): relative Frobenius <= 2e-2.
"""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GRIDS = [(1, 1, False), (1, 2, True), (2, 1, False), (2, 2, False)]


@pytest.fixture(scope="module")
def tess():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2105_14500_b200 as t
    return t


def f32r(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def bf16r(a):
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    # round-to-nearest-even to the top 16 bits
    u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def rel_diff(v, r):
    return np.abs(v - r).max() / max(np.abs(r).max(), 1e-30)


def frob(v, r):
    return np.linalg.norm(v - r) / max(np.linalg.norm(r), 1e-30)


@pytest.mark.parametrize("q,d,allow", GRIDS)
def test_config1_nn_fp32(tess, orc, q, d, allow):
    # BASELINE.json config 1: A, B 1024x1024, streams (42,0), (42,1), fp32.
    a = f32r(orc.random_matrix(1024, 1024, 42, 0))
    b = f32r(orc.random_matrix(1024, 1024, 42, 1))
    want, sr, sk = orc.tesseract_matmul(a, b, q, d, "nn")
    got = tess.tesseract_matmul(a, b, tess.GridSpec(q, d, allow), "nn", dtype="f32")
    assert rel_diff(got.value, want) <= 1e-5
    assert (got.stats.per_rank == sr).all() and (got.stats.per_kind == sk).all()


@pytest.mark.parametrize("q,d,allow", GRIDS + [(3, 1, False)])
@pytest.mark.parametrize("variant", ["nn", "nt", "tn"])
def test_variants_fp32(tess, orc, q, d, allow, variant):
    m, n, r = 48 * q * d, 40 * q, 24 * q
    a = f32r(orc.random_matrix(m, n, 5, 0))
    b = f32r(orc.random_matrix({"nn": n, "nt": r, "tn": m}[variant],
                               {"nn": r, "nt": n, "tn": r}[variant], 5, 1))
    want, sr, sk = orc.tesseract_matmul(a, b, q, d, variant)
    got = tess.tesseract_matmul(a, b, tess.GridSpec(q, d, allow), variant, dtype="f32")
    assert rel_diff(got.value, want) <= 1e-5
    assert (got.stats.per_rank == sr).all() and (got.stats.per_kind == sk).all()


@pytest.mark.parametrize("q,d,allow", GRIDS)
@pytest.mark.parametrize("variant", ["nn", "nt", "tn"])
def test_variants_bf16(tess, orc, q, d, allow, variant):
    m, n, r = 256 * q * d, 256 * q, 128 * q
    a0 = orc.random_matrix(m, n, 6, 0)
    b0 = orc.random_matrix({"nn": n, "nt": r, "tn": m}[variant],
                           {"nn": r, "nt": n, "tn": r}[variant], 6, 1)
    a, b = bf16r(a0), bf16r(b0)
    want, sr, sk = orc.tesseract_matmul(a, b, q, d, variant)
    want0, _, _ = orc.tesseract_matmul(a0, b0, q, d, variant)
    got = tess.tesseract_matmul(a0, b0, tess.GridSpec(q, d, allow), variant, dtype="bf16")
    assert frob(got.value, want) <= 1e-4
    assert frob(got.value, want0) <= 5e-3
    assert (got.stats.per_rank == sr).all() and (got.stats.per_kind == sk).all()


@pytest.mark.parametrize("q,d,allow", GRIDS)
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_backward(tess, orc, q, d, allow, dtype):
    m, k, n = 128 * q * d, 64 * q, 96 * q
    rnd = f32r if dtype == "f32" else bf16r
    a = rnd(orc.random_matrix(m, k, 7, 0))
    b = rnd(orc.random_matrix(k, n, 7, 1))
    dc = rnd(orc.random_matrix(m, n, 7, 2))
    da, db, sr, sk = orc.tesseract_backward(dc, a, b, q, d)
    got = tess.tesseract_backward_dense(dc, a, b, tess.GridSpec(q, d, allow), dtype=dtype)
    if dtype == "f32":
        assert rel_diff(got.a_grad, da) <= 1e-5 and rel_diff(got.b_grad, db) <= 1e-5
    else:
        assert frob(got.a_grad, da) <= 1e-4 and frob(got.b_grad, db) <= 1e-4
    assert (got.stats.per_rank == sr).all() and (got.stats.per_kind == sk).all()


def test_partition_bit_exact(tess, orc):
    import torch
    q, d = 2, 2
    grid = tess.GridSpec(q, d)
    ctxs = tess.init_local(grid)
    try:
        m = orc.random_matrix(64, 48, 8, 0).astype(np.float32)
        gdev = torch.from_numpy(m).cuda()
        for scheme in (0, 1):
            blocks = orc.partition(m.astype(np.float64), q, d, scheme)
            back = torch.zeros_like(gdev)
            for r, cx in enumerate(ctxs):
                loc = torch.empty(blocks[r].shape, dtype=torch.float32, device="cuda")
                cx.partition(scheme, "f32", gdev.data_ptr(), 64, 48, loc.data_ptr())
                torch.cuda.synchronize()
                assert (loc.cpu().numpy().astype(np.float64) == blocks[r]).all()
                cx.unpartition(scheme, "f32", loc.data_ptr(), 64, 48, back.data_ptr())
            torch.cuda.synchronize()
            assert torch.equal(back, gdev)
        # bf16 bytes round-trip bit-exactly too
        gb = gdev.to(torch.bfloat16)
        back = torch.zeros_like(gb)
        for cx in ctxs:
            loc = torch.empty((64 // 4, 48 // 2), dtype=torch.bfloat16, device="cuda")
            cx.partition(0, "bf16", gb.data_ptr(), 64, 48, loc.data_ptr())
            cx.unpartition(0, "bf16", loc.data_ptr(), 64, 48, back.data_ptr())
        torch.cuda.synchronize()
        assert torch.equal(back.view(torch.int16), gb.view(torch.int16))
    finally:
        for cx in ctxs:
            cx.close()


def _layer_inputs(orc, b, s, h, seed, rnd):
    x = rnd(orc.random_matrix(b * s, h, seed, 0))
    dy = rnd(orc.random_matrix(b * s, h, seed, 2))
    P = orc.random_block_params(h, seed, 100)
    P = {k: (rnd(v) if k.startswith("w_") else f32r(v)) for k, v in P.items()}
    return x, dy, P


def _compare_layer(res, want, tol, metric):
    errs = {"y": metric(res.y, want["y"]), "dx": metric(res.dx, want["dx"])}
    for k, v in want["grads"].items():
        if np.abs(v).max() > 0:
            errs[k] = metric(res.grads[k], v)
        else:
            assert np.abs(res.grads[k]).max() == 0, k
    worst = max(errs.values())
    assert worst <= tol, errs


@pytest.mark.parametrize("q,d,allow", GRIDS)
@pytest.mark.parametrize("op", ["feedforward", "attention", "layernorm", "bias_add", "block"])
def test_layers_fp32(tess, orc, q, d, allow, op):
    b, s, h, nh = 4, 8, 32, 4
    x, dy, P = _layer_inputs(orc, b, s, h, 9, f32r)
    want = orc.layer_run(op, x, dy, P, b, s, nh)
    res = tess.layer_run(op, x, dy, P, tess.LayerDims(b, s, h, nh), tess.GridSpec(q, d, allow),
                         dtype="f32")
    _compare_layer(res, want, 1e-5, rel_diff)
    if op == "bias_add":
        assert rel_diff(res.dbias, want["dbias"]) <= 1e-5
    sr, sk = orc.layer_stats(op, q, d, b, s, h)
    assert (res.stats.per_rank == sr).all() and (res.stats.per_kind == sk).all()


@pytest.mark.parametrize("q,d,allow", GRIDS)
@pytest.mark.parametrize("op", ["feedforward", "attention", "layernorm", "block"])
def test_layers_bf16(tess, orc, q, d, allow, op):
    b, s, h, nh = 4, 64, 128, 4
    x, dy, P = _layer_inputs(orc, b, s, h, 10, bf16r)
    want = orc.layer_run(op, x, dy, P, b, s, nh)
    res = tess.layer_run(op, x, dy, P, tess.LayerDims(b, s, h, nh), tess.GridSpec(q, d, allow),
                         dtype="bf16")
    _compare_layer(res, want, 2e-2, frob)
    sr, sk = orc.layer_stats(op, q, d, b, s, h)
    assert (res.stats.per_rank == sr).all() and (res.stats.per_kind == sk).all()


def test_error_taxonomy(tess, orc):
    a = orc.random_matrix(8, 6, 1, 0)
    with pytest.raises(tess.ShapeError):
        tess.tesseract_matmul(a, orc.random_matrix(5, 4, 1, 1), tess.GridSpec(1, 1))
    with pytest.raises(tess.DivisibilityError, match="rows"):
        tess.tesseract_matmul(orc.random_matrix(6, 4, 1, 0), orc.random_matrix(4, 4, 1, 1),
                              tess.GridSpec(2, 2))
    with pytest.raises(tess.DivisibilityError, match="batch"):
        x = orc.random_matrix(3 * 2, 8, 1, 0)
        P = orc.random_block_params(8, 1, 100)
        tess.layer_run("block", x, x, P, tess.LayerDims(3, 2, 8, 2), tess.GridSpec(2, 1))


def test_determinism_bitwise(tess, orc):
    a = orc.random_matrix(256, 128, 3, 0)
    b = orc.random_matrix(128, 192, 3, 1)
    g = tess.GridSpec(2, 2)
    r1 = tess.tesseract_matmul(a, b, g, "nn", dtype="bf16").value
    r2 = tess.tesseract_matmul(a, b, g, "nn", dtype="bf16").value
    assert (r1 == r2).all()


def test_degeneracy_summa_equals_tesseract_d1(tess, orc):
    # [q,q,1] Tesseract == SUMMA in values and CommStats.
    a = f32r(orc.random_matrix(96, 64, 4, 0))
    b = f32r(orc.random_matrix(64, 80, 4, 1))
    got = tess.tesseract_matmul(a, b, tess.GridSpec(2, 1), "nn")
    want, sr, sk = orc.tesseract_matmul(a, b, 2, 1, "nn")
    assert rel_diff(got.value, want) <= 1e-5 and (got.stats.per_kind == sk).all()


def test_per_rank_contexts_threaded_nn(tess, orc):
    """Drive the per-rank C-ABI from one Python thread per rank (run_spmd)."""
    import torch
    q, d = 2, 2
    grid = tess.GridSpec(q, d)
    M, K, N = 128, 96, 64
    a = f32r(orc.random_matrix(M, K, 12, 0))
    b = f32r(orc.random_matrix(K, N, 12, 1))
    want, _, sk = orc.tesseract_matmul(a, b, q, d, "nn")
    ab = orc.partition(a, q, d, 0)
    bb = orc.partition(b, q, d, 1)
    ctxs = tess.init_local(grid)
    outs = [None] * grid.size()
    errs = []

    def run(r):
        try:
            cx = ctxs[r]
            la = torch.from_numpy(ab[r].astype(np.float32)).cuda()
            lb = torch.from_numpy(bb[r].astype(np.float32)).cuda()
            lc = torch.empty((la.shape[0], lb.shape[1]), dtype=torch.float32, device="cuda")
            cx.matmul("nn", "f32", la.data_ptr(), *la.shape, lb.data_ptr(), *lb.shape,
                      lc.data_ptr())
            torch.cuda.synchronize()
            outs[r] = lc.cpu().numpy().astype(np.float64)
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=run, args=(r,)) for r in range(grid.size())]
    [t.start() for t in th]
    [t.join() for t in th]
    try:
        assert not errs, errs
        got = orc.combine(outs, M, N, q, d, 0)
        assert rel_diff(got, want) <= 1e-5
        assert sum(cx.stats()["by_kind"][0][0] for cx in ctxs) == int(sk[0, 0])
    finally:
        for cx in ctxs:
            cx.close()


@pytest.mark.parametrize("q,d,allow", [(2, 2, False), (1, 2, True), (1, 1, False)])
def test_train_toy_fp32_tracks_reference(tess, orc, q, d, allow):
    # ToyConfig defaults (layers.hpp:256): dims {4,4,8,2}, 2 layers, lr 0.05, seed 1234
    b, s, h, nh, L, steps, lr, seed = 4, 4, 8, 2, 2, 12, 0.05, 1234
    want = orc.train_toy(b, s, h, nh, L, steps, lr, seed)
    x = f32r(orc.random_matrix(b * s, h, seed, 0))
    tgt = f32r(orc.random_matrix(b * s, h, seed, 1))
    P = [{k: f32r(v) for k, v in orc.random_block_params(h, seed, 100 + l).items()}
         for l in range(L)]
    res = tess.train_toy(tess.LayerDims(b, s, h, nh), L, steps, lr, tess.GridSpec(q, d, allow),
                         x, tgt, P, dtype="f32")
    assert np.abs(res.dist_loss - want).max() / want.max() <= 1e-5, (res.dist_loss, want)
    assert res.dist_loss[-1] < res.dist_loss[0]  # it trains


def test_train_toy_bf16(tess, orc):
    b, s, h, nh, L, steps, lr, seed = 4, 64, 128, 4, 2, 4, 0.05, 99
    want = orc.train_toy(b, s, h, nh, L, steps, lr, seed)
    x = orc.random_matrix(b * s, h, seed, 0)
    tgt = orc.random_matrix(b * s, h, seed, 1)
    P = [orc.random_block_params(h, seed, 100 + l) for l in range(L)]
    res = tess.train_toy(tess.LayerDims(b, s, h, nh), L, steps, lr, tess.GridSpec(2, 2), x, tgt,
                         P, dtype="bf16")
    assert np.abs(res.dist_loss - want).max() / want.max() <= 2e-2, (res.dist_loss, want)


@pytest.mark.parametrize("p", [1, 2, 4, 8])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_megatron_1d_linear(tess, orc, p, dtype):
    rnd = f32r if dtype == "f32" else bf16r
    x = rnd(orc.random_matrix(64, 128, 15, 0))
    w1 = rnd(orc.random_matrix(128, 256, 15, 1))
    w2 = rnd(orc.random_matrix(256, 96, 15, 2))
    want = orc.megatron_1d_linear(x, w1, w2, p)
    got = tess.megatron_1d_linear(x, w1, w2, p, dtype=dtype)
    if dtype == "f32":
        assert rel_diff(got.value, want) <= 1e-5
    else:  # the X W1_k intermediate is stored in bf16 between the two GEMMs
        assert frob(got.value, want) <= 1e-2
    # one all-reduce of [64, 96] over the p-rank line (flat counting)
    assert got.stats.by_kind("all_reduce") == ((2 * (p - 1), 2 * (p - 1) * 64 * 96) if p > 1
                                               else (0, 0))


def test_summa_is_tesseract_d1(tess, orc):
    a = f32r(orc.random_matrix(96, 64, 16, 0))
    b = f32r(orc.random_matrix(64, 80, 16, 1))
    want, _, sk = orc.tesseract_matmul(a, b, 2, 1, "nn")
    got = tess.summa_matmul(a, b, 2)
    assert rel_diff(got.value, want) <= 1e-5 and (got.stats.per_kind == sk).all()


def test_nccl_backend_world1_matches_local(tess, orc):
    """The NCCL backend (dlopen'd libnccl, world communicator + the three
    ncclCommSplits with NCCL_SPLIT_NOCOLOR for single-member groups) on a
    [1,1,1] grid runs a bf16 Transformer block bitwise like the in-process
    backend. (NCCL refuses two ranks on one GPU, so N>1 data movement is
    covered by the in-process backend on every grid instead.)"""
    import torch
    b, s, h, nh = 2, 64, 128, 2
    x, dy, P = _layer_inputs(orc, b, s, h, 11, bf16r)
    dev = torch.device("cuda", 0)
    bf = torch.bfloat16
    names = ("w_qkv", "w_proj", "w_ff1", "w_ff2")
    W = [torch.tensor(P[k], dtype=torch.float32, device=dev).to(bf).contiguous() for k in names]
    LN = [torch.tensor(P[k], dtype=torch.float32, device=dev).contiguous()
          for k in ("ln1_gain", "ln1_bias", "ln2_gain", "ln2_bias")]
    xt = torch.tensor(x, dtype=torch.float32, device=dev).to(bf)
    dyt = torch.tensor(dy, dtype=torch.float32, device=dev).to(bf)
    shard = tess.BlockShardC(*[t.data_ptr() for t in W + LN], 1e-5)
    dims = tess.LayerDims(b, s, h, nh)
    st = torch.cuda.current_stream().cuda_stream
    outs = []
    for kind in ("local", "nccl"):
        ctx = (tess.init_local(tess.GridSpec(1, 1))[0] if kind == "local" else
               tess.init_nccl(tess.GridSpec(1, 1), 0, 0, tess.nccl_unique_id()))
        try:
            y, dx = torch.empty_like(xt), torch.empty_like(xt)
            G = [torch.zeros(t.shape, device=dev) for t in W + LN]
            grads = tess.BlockGradsC(*[t.data_ptr() for t in G])
            ctx.layer_forward("block", "bf16", dims, shard, xt.data_ptr(), y.data_ptr(), stream=st)
            ctx.layer_backward("block", "bf16", dims, shard, dyt.data_ptr(), dx.data_ptr(), grads,
                               stream=st)
            torch.cuda.synchronize()
            ctx.barrier()
            outs.append([y.clone(), dx.clone()] + [g.clone() for g in G])
        finally:
            ctx.close()
    for a, c in zip(*outs):
        assert torch.equal(a, c)


def test_comm_noop_keeps_schedule_and_meter(tess, orc):
    """tess_set_comm_noop (bench.py's exposed-communication measurement): the
    [2,2,2] NN product runs through the same schedule with no data moved --
    identical CommStats, and switching it off restores the exact result."""
    import torch
    q, d = 2, 2
    grid = tess.GridSpec(q, d)
    M, K, N = 128, 96, 64
    a = f32r(orc.random_matrix(M, K, 13, 0))
    b = f32r(orc.random_matrix(K, N, 13, 1))
    want, _, _ = orc.tesseract_matmul(a, b, q, d, "nn")
    ab = orc.partition(a, q, d, 0)
    bb = orc.partition(b, q, d, 1)
    ctxs = tess.init_local(grid)
    outs = [None] * grid.size()
    stats = {}
    errs = []

    def run(r, noop):
        try:
            cx = ctxs[r]
            cx.set_comm_noop(noop)
            cx.reset_stats()
            la = torch.from_numpy(ab[r].astype(np.float32)).cuda()
            lb = torch.from_numpy(bb[r].astype(np.float32)).cuda()
            lc = torch.zeros((la.shape[0], lb.shape[1]), dtype=torch.float32, device="cuda")
            cx.matmul("nn", "f32", la.data_ptr(), *la.shape, lb.data_ptr(), *lb.shape,
                      lc.data_ptr())
            torch.cuda.synchronize()
            outs[r] = lc.cpu().numpy().astype(np.float64)
            stats[(noop, r)] = cx.stats()["by_kind"]
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    try:
        for noop in (True, False):
            th = [threading.Thread(target=run, args=(r, noop)) for r in range(grid.size())]
            [t.start() for t in th]
            [t.join() for t in th]
            assert not errs, errs
        got = orc.combine(outs, M, N, q, d, 0)
        assert rel_diff(got, want) <= 1e-5
        for r in range(grid.size()):
            assert stats[(True, r)] == stats[(False, r)]
    finally:
        for cx in ctxs:
            cx.close()


@pytest.mark.parametrize("q,d,allow", [(1, 1, False), (1, 2, True)])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_layernorm_fused_single_pass(tess, orc, q, d, allow, dtype):
    """hidden/q a multiple of 4096 with a one-member row group: the fused
    single-pass LayerNorm kernels (stats + apply; stats + dx + dgain/dbias)
    against the fp64 oracle."""
    b, s, h, nh = 2, 8, 4096, 32
    rnd = f32r if dtype == "f32" else bf16r
    x, dy, P = _layer_inputs(orc, b, s, h, 17, rnd)
    want = orc.layer_run("layernorm", x, dy, P, b, s, nh)
    res = tess.layer_run("layernorm", x, dy, P, tess.LayerDims(b, s, h, nh),
                         tess.GridSpec(q, d, allow), dtype=dtype)
    if dtype == "f32":
        _compare_layer(res, want, 1e-5, rel_diff)
    else:
        _compare_layer(res, want, 2e-2, frob)
    sr, sk = orc.layer_stats("layernorm", q, d, b, s, h)
    assert (res.stats.per_rank == sr).all() and (res.stats.per_kind == sk).all()


@pytest.mark.parametrize("h", [8192, 12288])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_layernorm_fused_vs_torch(tess, h, dtype):
    """The fused LayerNorm at the wider hidden sizes (two and three 4096-column
    passes per thread; 12288 is cfg4's) against torch fp32 LayerNorm fwd+bwd
    (eps 1e-5, ref layers.hpp:48) on the same rounded inputs."""
    import torch
    torch.manual_seed(1)
    dev = torch.device("cuda", 0)
    rows = 64
    tdt = torch.float32 if dtype == "f32" else torch.bfloat16
    x = torch.randn(rows, h, device=dev).to(tdt)
    dy = torch.randn(rows, h, device=dev).to(tdt)
    gain = (1 + 0.1 * torch.randn(h, device=dev)).float()
    bias = (0.1 * torch.randn(h, device=dev)).float()
    ctx = tess.init_local(tess.GridSpec(1, 1))[0]
    try:
        dummy = torch.zeros(8, device=dev, dtype=tdt)
        shard = tess.BlockShardC(*[dummy.data_ptr()] * 4, gain.data_ptr(), bias.data_ptr(),
                                 gain.data_ptr(), bias.data_ptr(), 1e-5)
        G = [torch.zeros(8, device=dev) for _ in range(4)] + \
            [torch.zeros(h, device=dev) for _ in range(4)]
        grads = tess.BlockGradsC(*[t.data_ptr() for t in G])
        y, dx = torch.empty_like(x), torch.empty_like(x)
        dims = tess.LayerDims(1, rows, h, 32)
        st = torch.cuda.current_stream().cuda_stream
        ctx.layer_forward("layernorm", dtype, dims, shard, x.data_ptr(), y.data_ptr(), stream=st)
        ctx.layer_backward("layernorm", dtype, dims, shard, dy.data_ptr(), dx.data_ptr(), grads,
                           stream=st)
        torch.cuda.synchronize()
    finally:
        ctx.close()
    xr = x.float().requires_grad_(True)
    g_, b_ = gain.clone().requires_grad_(True), bias.clone().requires_grad_(True)
    yr = torch.nn.functional.layer_norm(xr, (h,), g_, b_, eps=1e-5)
    yr.backward(dy.float())
    tol = 1e-5 if dtype == "f32" else 1e-2

    def rel(a, r):
        return ((a.float() - r).norm() / r.norm()).item()
    errs = {"y": rel(y, yr.detach()), "dx": rel(dx, xr.grad), "dgain": rel(G[4], g_.grad),
            "dbias": rel(G[5], b_.grad)}
    assert max(errs.values()) <= tol, errs


def test_block_fused_layernorm_bf16(tess, orc):
    b, s, h, nh = 1, 8, 4096, 32
    x, dy, P = _layer_inputs(orc, b, s, h, 18, bf16r)
    want = orc.layer_run("block", x, dy, P, b, s, nh)
    res = tess.layer_run("block", x, dy, P, tess.LayerDims(b, s, h, nh), tess.GridSpec(1, 1),
                         dtype="bf16")
    _compare_layer(res, want, 2e-2, frob)


@pytest.mark.parametrize("variant", ["nn", "nt", "tn"])
@pytest.mark.parametrize("out", ["bf16", "f32", "f32_accumulate"])
def test_gemm_ragged_wide_tiles(tess, variant, out):
    """Ragged M, N, K (not multiples of the 256 x 512 pair tile or the 64-deep
    k-block) on shapes the dispatcher routes to the 256 x 512 pair kernel with
    the TMA-store / TMA-reduce-add epilogue and the dynamic tile schedule,
    against a torch fp32 product of the same bf16 inputs."""
    import torch
    torch.manual_seed(7)
    dev = torch.device("cuda", 0)
    M, N, K = 2000, 2600, 1000
    bf = torch.bfloat16
    if variant == "nn":
        a, b = torch.randn(M, K, device=dev, dtype=bf), torch.randn(K, N, device=dev, dtype=bf)
        ref = a.float() @ b.float()
        dims = (M, K, K, N)
    elif variant == "nt":
        a, b = torch.randn(M, K, device=dev, dtype=bf), torch.randn(N, K, device=dev, dtype=bf)
        ref = a.float() @ b.float().t()
        dims = (M, K, N, K)
    else:
        a, b = torch.randn(K, M, device=dev, dtype=bf), torch.randn(K, N, device=dev, dtype=bf)
        ref = a.float().t() @ b.float()
        dims = (K, M, K, N)
    acc = out == "f32_accumulate"
    ctype = "bf16" if out == "bf16" else "f32"
    c = (torch.randn(M, N, device=dev) if acc else
         torch.zeros(M, N, device=dev, dtype=bf if out == "bf16" else torch.float32))
    c0 = c.clone()
    ctx = tess.init_local(tess.GridSpec(1, 1))[0]
    try:
        ctx.matmul(variant, "bf16", a.data_ptr(), dims[0], dims[1], b.data_ptr(), dims[2],
                   dims[3], c.data_ptr(), c_dtype=ctype, accumulate=acc,
                   stream=torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
    finally:
        ctx.close()
    want = ref + c0 if acc else ref
    err = ((c.float() - want).norm() / want.norm()).item()
    assert err <= (5e-3 if out == "bf16" else 1e-5), err


def test_layer_step_matches_forward_backward_host_buffers(tess, orc):
    """tess_layer_step (x and dy together; a host dy uploads while the forward
    runs) gives bitwise the results of tess_layer_forward +
    tess_layer_backward, with pinned host inputs/outputs; a host output fed
    back as the next input is ordered after its pending copy."""
    import torch
    b, s, h, nh = 2, 64, 256, 2
    x, dy, P = _layer_inputs(orc, b, s, h, 19, bf16r)
    dev = torch.device("cuda", 0)
    bf = torch.bfloat16
    names = ("w_qkv", "w_proj", "w_ff1", "w_ff2")
    W = [torch.tensor(P[k], dtype=torch.float32, device=dev).to(bf).contiguous() for k in names]
    LN = [torch.tensor(P[k], dtype=torch.float32, device=dev).contiguous()
          for k in ("ln1_gain", "ln1_bias", "ln2_gain", "ln2_bias")]
    xh = torch.tensor(x, dtype=torch.float32).to(bf).pin_memory()
    dyh = torch.tensor(dy, dtype=torch.float32).to(bf).pin_memory()
    shard = tess.BlockShardC(*[t.data_ptr() for t in W + LN], 1e-5)
    dims = tess.LayerDims(b, s, h, nh)
    st = torch.cuda.current_stream().cuda_stream
    outs = []
    for mode in ("split", "step"):
        ctx = tess.init_local(tess.GridSpec(1, 1))[0]
        try:
            yh, dxh = torch.empty_like(xh).pin_memory(), torch.empty_like(xh).pin_memory()
            G = [torch.zeros(t.shape, device=dev) for t in W + LN]
            grads = tess.BlockGradsC(*[t.data_ptr() for t in G])
            for _ in range(2):
                src = xh
                if mode == "split":
                    ctx.layer_forward("block", "bf16", dims, shard, src.data_ptr(), yh.data_ptr(),
                                      stream=st)
                    ctx.layer_backward("block", "bf16", dims, shard, dyh.data_ptr(),
                                       dxh.data_ptr(), grads, stream=st)
                else:
                    ctx.layer_step("block", "bf16", dims, shard, src.data_ptr(), dyh.data_ptr(),
                                   yh.data_ptr(), dxh.data_ptr(), grads, stream=st)
            # chained: the host output y fed back as the next input
            if mode == "split":
                ctx.layer_forward("block", "bf16", dims, shard, yh.data_ptr(), dxh.data_ptr(),
                                  stream=st)
                ctx.layer_backward("block", "bf16", dims, shard, dyh.data_ptr(), yh.data_ptr(),
                                   grads, stream=st)
            else:
                ctx.layer_step("block", "bf16", dims, shard, yh.data_ptr(), dyh.data_ptr(),
                               dxh.data_ptr(), yh.data_ptr(), grads, stream=st)
            ctx.stream_join(st)
            torch.cuda.synchronize()
            outs.append([yh.clone(), dxh.clone()] + [g.cpu() for g in G])
        finally:
            ctx.close()
    for a, c in zip(*outs):
        assert torch.equal(a, c)


def test_layer_step_distinct_inputs_per_step(tess, orc):
    """Four consecutive tess_layer_step calls with different pinned host x / dy
    each step (the per-call double-buffered upload staging, reused every
    second call) give bitwise the outputs and accumulated gradients of
    tess_layer_forward + tess_layer_backward on the same sequence."""
    import torch
    b, s, h, nh = 2, 64, 256, 2
    _, _, P = _layer_inputs(orc, b, s, h, 23, bf16r)
    dev = torch.device("cuda", 0)
    bf = torch.bfloat16
    names = ("w_qkv", "w_proj", "w_ff1", "w_ff2")
    W = [torch.tensor(P[k], dtype=torch.float32, device=dev).to(bf).contiguous() for k in names]
    LN = [torch.tensor(P[k], dtype=torch.float32, device=dev).contiguous()
          for k in ("ln1_gain", "ln1_bias", "ln2_gain", "ln2_bias")]
    steps = 4
    xs = [torch.tensor(bf16r(orc.random_matrix(b * s, h, 30 + k, 0)), dtype=torch.float32)
          .to(bf).pin_memory() for k in range(steps)]
    dys = [torch.tensor(bf16r(orc.random_matrix(b * s, h, 30 + k, 2)), dtype=torch.float32)
           .to(bf).pin_memory() for k in range(steps)]
    shard = tess.BlockShardC(*[t.data_ptr() for t in W + LN], 1e-5)
    dims = tess.LayerDims(b, s, h, nh)
    st = torch.cuda.current_stream().cuda_stream
    outs = []
    for mode in ("split", "step"):
        ctx = tess.init_local(tess.GridSpec(1, 1))[0]
        try:
            ys = [torch.empty_like(xs[0]).pin_memory() for _ in range(steps)]
            dxs = [torch.empty_like(xs[0]).pin_memory() for _ in range(steps)]
            G = [torch.zeros(t.shape, device=dev) for t in W + LN]
            grads = tess.BlockGradsC(*[t.data_ptr() for t in G])
            for k in range(steps):
                if mode == "split":
                    ctx.layer_forward("block", "bf16", dims, shard, xs[k].data_ptr(),
                                      ys[k].data_ptr(), stream=st)
                    ctx.layer_backward("block", "bf16", dims, shard, dys[k].data_ptr(),
                                       dxs[k].data_ptr(), grads, stream=st)
                else:
                    ctx.layer_step("block", "bf16", dims, shard, xs[k].data_ptr(),
                                   dys[k].data_ptr(), ys[k].data_ptr(), dxs[k].data_ptr(), grads,
                                   stream=st)
            ctx.stream_join(st)
            torch.cuda.synchronize()
            outs.append([t.clone() for t in ys + dxs] + [g.cpu() for g in G])
        finally:
            ctx.close()
    for a, c in zip(*outs):
        assert torch.equal(a, c)
    assert not torch.equal(outs[0][0], outs[0][1])  # the steps really differ


@pytest.mark.parametrize("offset,outlier", [(0.0, 0.0), (1000.0, 0.0), (0.0, 3000.0),
                                            (-250.0, 4000.0)])
def test_layernorm_fused_offset_rows_fp32(tess, offset, outlier):
    """The fused single-pass LayerNorm (per-thread mean / M2 combined by Chan's
    formula) on rows whose mean is far from zero or whose first element is
    an outlier, against the fp64 LayerNorm of the same fp32 inputs
    (reference layers.cpp:242-281 with hidden_total = h): no cancellation."""
    import torch
    h, rows = 12288, 32
    g = torch.Generator().manual_seed(3)
    x = (offset + torch.randn(rows, h, generator=g, dtype=torch.float64)).float()
    x[:, 0] += outlier
    gain = torch.ones(h)
    bias = torch.zeros(h)
    dev = torch.device("cuda", 0)
    xd = x.to(dev)
    gd, bd = gain.to(dev), bias.to(dev)
    ctx = tess.init_local(tess.GridSpec(1, 1))[0]
    try:
        dummy = torch.zeros(8, device=dev)
        shard = tess.BlockShardC(*[dummy.data_ptr()] * 4, gd.data_ptr(), bd.data_ptr(),
                                 gd.data_ptr(), bd.data_ptr(), 1e-5)
        y = torch.empty_like(xd)
        ctx.layer_forward("layernorm", "f32", tess.LayerDims(1, rows, h, 32), shard,
                          xd.data_ptr(), y.data_ptr(),
                          stream=torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
    finally:
        ctx.close()
    xf = x.double()
    mu = xf.mean(1, keepdim=True)
    var = ((xf - mu) ** 2).mean(1, keepdim=True)
    want = (xf - mu) / torch.sqrt(var + 1e-5)
    err = ((y.cpu().double() - want).norm() / want.norm()).item()
    assert err <= 1e-4, err


@pytest.mark.parametrize("q,d,allow", GRIDS)
@pytest.mark.parametrize("h", [2048, 12288])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_layernorm_vectorised_widths(tess, orc, q, d, allow, h, dtype):
    """The vectorised LayerNorm at widths h/q of the configs: 12288/2 = 6144
    (cfg4 on q = 2: 768-thread blocks, one pass), 2048 and 1024 (256- and
    128-thread blocks); q = 1 runs the fused single pass, q = 2 the split
    partials -> row all-reduce -> apply (forward) and partials + dgain/dbias
    -> all-reduce -> dx (backward). Against the fp64 oracle
    (layers.cpp:242-345), CommStats equal."""
    b, s, nh = 2 * q * d, 4, 16
    rnd = f32r if dtype == "f32" else bf16r
    x, dy, P = _layer_inputs(orc, b, s, h, 27, rnd)
    want = orc.layer_run("layernorm", x, dy, P, b, s, nh)
    tess.profile_enable(True)
    try:
        res = tess.layer_run("layernorm", x, dy, P, tess.LayerDims(b, s, h, nh),
                             tess.GridSpec(q, d, allow), dtype=dtype)
        kernels = tess.profile_kernels()
    finally:
        tess.profile_enable(False)
    if dtype == "f32":
        _compare_layer(res, want, 1e-5, rel_diff)
    else:
        _compare_layer(res, want, 2e-2, frob)
    sr, sk = orc.layer_stats("layernorm", q, d, b, s, h)
    assert (res.stats.per_rank == sr).all() and (res.stats.per_kind == sk).all()
    want_k = {"ln_fused_fwd_kernel", "ln_fused_bwd_kernel"} if q == 1 else \
        {"ln_vec_stats_kernel", "ln_vec_apply_kernel", "ln_vec_bwd_stats_kernel",
         "ln_vec_bwd_apply_kernel"}
    assert want_k <= set(kernels), sorted(kernels)


@pytest.mark.parametrize("q,d,allow", [(2, 1, False), (2, 2, False)])
def test_block_vectorised_layernorm_q2_bf16(tess, orc, q, d, allow):
    """A bf16 block on q = 2 grids with h/q = 1024 (vectorised split LayerNorm,
    128-thread blocks, residual folded into the backward apply)."""
    b, s, h, nh = 2 * q * d, 8, 2048, 16
    x, dy, P = _layer_inputs(orc, b, s, h, 28, bf16r)
    want = orc.layer_run("block", x, dy, P, b, s, nh)
    res = tess.layer_run("block", x, dy, P, tess.LayerDims(b, s, h, nh),
                         tess.GridSpec(q, d, allow), dtype="bf16")
    _compare_layer(res, want, 2e-2, frob)
