"""BASELINE config 5 at its real layer shape (24-layer stack of h=4096, s=2048,
b=16, 32 heads -- SURVEY 8d's proposal): the three schemes' communication per
GPU for one layer fwd+bwd, from the context meters (reference counting rules,
runtime.hpp:24-69), run in-process on ONE B200 (the ranks share the GPU, so
the wall times say nothing about scaling; the metered volumes are exact):
  Tesseract [2,2,2] (8 ranks), SUMMA [2,2] (= Tesseract [2,2,1], 4 ranks),
  Megatron 1-D [8] (tess_megatron_layer_run, 8 ranks).
Prints one JSON line per scheme. LAYERS scales the per-layer numbers to the
stack (every layer moves the same)."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (input generator only: the reference's RNG streams)
import paper_2105_14500_b200 as tess  # noqa: E402

b, s, h, nh = (int(v) for v in os.environ.get("SHAPE", "16,2048,4096,32").split(","))
LAYERS = int(os.environ.get("LAYERS", "24"))
orc = oracle.Oracle()
x = orc.random_matrix(b * s, h, 42, 0)
dy = orc.random_matrix(b * s, h, 42, 2)
P = orc.random_block_params(h, 42, 100)
dims = tess.LayerDims(b, s, h, nh)
T = b * s
flops = 72 * T * h * h + 12 * T * s * h


def report(name, ranks, res, sec):
    pr = np.asarray(res.stats.per_rank, dtype=np.float64)  # sent msgs, sent elems, recv msgs, recv elems
    line = {"scheme": name, "ranks": ranks, "layer_shape": {"b": b, "s": s, "h": h, "heads": nh},
            "per_gpu_sent_elements_max": int(pr[:, 1].max()),
            "per_gpu_recv_elements_max": int(pr[:, 3].max()),
            "per_gpu_recv_elements_x_layers": int(pr[:, 3].max()) * LAYERS,
            "by_kind": {k: list(res.stats.by_kind(k)) for k in tess.KIND_NAMES},
            "layer_flops": flops, "one_gpu_wall_s": round(sec, 2)}
    print(json.dumps(line), flush=True)


for name, ranks, run in [
    ("tesseract[2,2,2]", 8, lambda: tess.layer_run("block", x, dy, P, dims, tess.GridSpec(2, 2),
                                                   dtype="bf16")),
    ("summa[2,2]", 4, lambda: tess.layer_run("block", x, dy, P, dims, tess.GridSpec(2, 1),
                                             dtype="bf16")),
    ("megatron[8]", 8, lambda: tess.megatron_layer_run("block", x, dy, P, dims, 8, dtype="bf16")),
]:
    t0 = time.time()
    res = run()
    report(name, ranks, res, time.time() - t0)
    del res
