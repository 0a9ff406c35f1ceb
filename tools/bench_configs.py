"""BASELINE configs 2 and 3 on one B200 through the rank-level C-ABI ([1,1,1]):
  cfg2  Tesseract Linear fwd+bwd: Y = X W (NN), dX = dY W^T (NT), dW = X^T dY (TN)
        X [16384 x 4096], W [4096 x 16384], bf16 -- 6*M*K*N flops
  cfg3  MLP block + distributed LayerNorm (LN2 -> FF1+GeLU -> FF2 -> +residual),
        h = 8192, s = 2048, b = 16 / 8 per GPU-equivalent of [2,2,2]: here the
        whole b = 2 share of one GPU of the 8 (T = 4096 tokens) -- 48*T*h^2 flops
Each: 3 warm-ups, 10 timed iterations (CUDA events). Prints one JSON line each."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2105_14500_b200 as tess  # noqa: E402


def timed(fn, warm=3, iters=10):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def main():
    dev = torch.device("cuda", 0)
    bf = torch.bfloat16
    st = torch.cuda.current_stream().cuda_stream
    ctx = tess.init_local(tess.GridSpec(1, 1))[0]
    # ---- cfg2
    M, K, N = 16384, 4096, 16384
    X = torch.randn(M, K, device=dev, dtype=bf)
    W = torch.randn(K, N, device=dev, dtype=bf) * K ** -0.5
    dY = torch.randn(M, N, device=dev, dtype=bf)
    Y = torch.empty(M, N, device=dev, dtype=bf)
    dX = torch.empty(M, K, device=dev, dtype=torch.float32)
    dW = torch.empty(K, N, device=dev, dtype=torch.float32)

    def linear():
        ctx.matmul("nn", "bf16", X.data_ptr(), M, K, W.data_ptr(), K, N, Y.data_ptr(),
                   c_dtype="bf16", stream=st)
        ctx.matmul("nt", "bf16", dY.data_ptr(), M, N, W.data_ptr(), K, N, dX.data_ptr(),
                   stream=st)
        ctx.matmul("tn", "bf16", X.data_ptr(), M, K, dY.data_ptr(), M, N, dW.data_ptr(),
                   sum_over_depth=True, stream=st)
    ms = timed(linear)
    print(json.dumps({"config": "cfg2 Linear fwd+bwd [1,1,1]", "M": M, "K": K, "N": N,
                      "ms": ms, "tflops": 6.0 * M * K * N / ms / 1e9}), flush=True)
    del X, W, dY, Y, dX, dW
    torch.cuda.empty_cache()
    # ---- cfg3 (MLP block incl. LayerNorm: layer op "feedforward" is the FF
    # alone; the block's MLP half = LN2 + FF + residual, timed via the FF op
    # plus a LayerNorm op on the same activations)
    h, s, b = 8192, 2048, 2
    T = b * s
    Wff = [torch.randn(sh, device=dev, dtype=bf) * h ** -0.5 for sh in ((h, 4 * h), (4 * h, h))]
    dummy = torch.zeros(8, device=dev, dtype=bf)
    LN = [torch.ones(h, device=dev), torch.zeros(h, device=dev)] * 2
    shard = tess.BlockShardC(dummy.data_ptr(), dummy.data_ptr(), Wff[0].data_ptr(),
                             Wff[1].data_ptr(), *[t.data_ptr() for t in LN], 1e-5)
    G = [torch.zeros(8, device=dev), torch.zeros(8, device=dev),
         torch.zeros(h, 4 * h, device=dev), torch.zeros(4 * h, h, device=dev)] + \
        [torch.zeros(h, device=dev) for _ in range(4)]
    grads = tess.BlockGradsC(*[t.data_ptr() for t in G])
    x = torch.randn(T, h, device=dev, dtype=bf)
    dy = torch.randn(T, h, device=dev, dtype=bf)
    y = torch.empty_like(x)
    ln = torch.empty_like(x)
    dx = torch.empty_like(x)
    dln = torch.empty_like(x)
    dims = tess.LayerDims(b, s, h, 64)

    def mlp():
        ctx.layer_forward("layernorm", "bf16", dims, shard, x.data_ptr(), ln.data_ptr(), stream=st)
        ctx.layer_forward("feedforward", "bf16", dims, shard, ln.data_ptr(), y.data_ptr(),
                          stream=st)
        ctx.layer_backward("feedforward", "bf16", dims, shard, dy.data_ptr(), dln.data_ptr(),
                           grads, stream=st)
        ctx.layer_backward("layernorm", "bf16", dims, shard, dln.data_ptr(), dx.data_ptr(),
                           grads, stream=st)
    ms = timed(mlp)
    print(json.dumps({"config": "cfg3 MLP + LayerNorm fwd+bwd [1,1,1] (one GPU's share of "
                                "[2,2,2]: b=2 of 16)", "T": T, "h": h, "ms": ms,
                      "tflops": 48.0 * T * h * h / ms / 1e9}), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
