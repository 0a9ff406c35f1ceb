"""Times the tess tcgen05 GEMM (through the C-ABI, tess_matmul on a [1,1,1]
context = one local GEMM) against cuBLAS (torch.matmul) on the cfg4 layer's
GEMM shapes, interleaved so both see the same clocks. Prints one JSON line
per shape."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2105_14500_b200 as tess  # noqa: E402

T, H = 8192, 12288
SHAPES = [  # name, variant, (a_rows, a_cols), (b_rows, b_cols)
    ("qkv_fwd_nn", "nn", (T, H), (H, 3 * H)),
    ("ff1_fwd_nn", "nn", (T, H), (H, 4 * H)),
    ("ff2_fwd_nn", "nn", (T, 4 * H), (4 * H, H)),
    ("ff2_dgrad_nt", "nt", (T, H), (4 * H, H)),
    ("ff1_wgrad_tn", "tn", (T, H), (T, 4 * H)),
]


def main():
    dev = torch.device("cuda", 0)
    ctx = tess.init_local(tess.GridSpec(1, 1))[0]
    iters = int(os.environ.get("ITERS", "5"))
    print("init ok", flush=True, file=sys.stderr)
    for name, v, sa, sb in SHAPES:
        print("shape", name, flush=True, file=sys.stderr)
        a = torch.randn(sa, device=dev, dtype=torch.bfloat16)
        b = torch.randn(sb, device=dev, dtype=torch.bfloat16)
        if v == "nn":
            M, N, K = sa[0], sb[1], sa[1]
            ref = lambda: a @ b  # noqa: E731
        elif v == "nt":
            M, N, K = sa[0], sb[0], sa[1]
            ref = lambda: a @ b.t()  # noqa: E731
        else:
            M, N, K = sa[1], sb[1], sa[0]
            ref = lambda: a.t() @ b  # noqa: E731
        c = torch.empty((M, N), device=dev, dtype=torch.bfloat16)
        st = torch.cuda.current_stream().cuda_stream

        def ours():
            ctx.matmul(v, "bf16", a.data_ptr(), *sa, b.data_ptr(), *sb, c.data_ptr(),
                       c_dtype="bf16", stream=st)

        def timeit(fn):
            for _ in range(2):
                fn()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(iters):
                fn()
            e1.record()
            torch.cuda.synchronize()
            return e0.elapsed_time(e1) / iters

        ours()
        torch.cuda.synchronize()
        print("first ours ok", flush=True, file=sys.stderr)
        res = {"shape": name, "M": M, "N": N, "K": K}
        for rnd in range(2):
            for label, fn in (("tess", ours), ("cublas", ref)):
                ms = timeit(fn)
                res[f"{label}_tflops_{rnd}"] = 2.0 * M * N * K / ms / 1e9
        ours()
        torch.cuda.synchronize()
        r = ref().float()
        cf = c.float()
        res["rel_frob_vs_cublas"] = ((cf - r).norm() / r.norm()).item()
        res["max_abs_diff"] = (cf - r).abs().max().item()
        res["frac_elems_differ"] = (cf != r).float().mean().item()
        print(json.dumps(res), flush=True)
        del a, b, c
        torch.cuda.empty_cache()
    ctx.close()


if __name__ == "__main__":
    main()
