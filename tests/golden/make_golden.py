"""Regenerates tests/golden/*.npz from the UNMODIFIED reference.

Run in the build container (where /root/reference exists) after
`make -C oracle ref`:  python tests/golden/make_golden.py

Every value is produced by oracle/_ref/libtsim_ref.so, i.e. the reference's
own tsim::tesseract_matmul / tesseract_backward_dense / layer_run /
random_block_params compiled from /root/reference/proj/src. The fixtures pin
the C restatement (oracle/tess_oracle.c) on machines where the reference
sources are absent (the GPU box).
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402

GRIDS = [(1, 1, False), (1, 2, True), (2, 1, False), (2, 2, False)]


def main():
    ref = oracle.Reference()
    out = {}
    # tesseract_matmul / backward on small seeded inputs (seed 11).
    for q, d, allow in GRIDS:
        m, n, r = 4 * q * d, 4 * q, 6 * q
        a = ref.random_matrix(m, n, 11, 0)
        for v, b in (("nn", ref.random_matrix(n, r, 11, 1)),
                     ("nt", ref.random_matrix(r, n, 11, 1)),
                     ("tn", ref.random_matrix(m, r, 11, 1))):
            c, sr, sk = ref.tesseract_matmul(a, b, q, d, v, allow=allow)
            key = f"mm_{v}_{q}{q}{d}"
            out[key + "_a"], out[key + "_b"], out[key + "_c"] = a, b, c
            out[key + "_sr"], out[key + "_sk"] = sr, sk
        k = 6 * q
        A = ref.random_matrix(m, k, 12, 0)
        B = ref.random_matrix(k, n, 12, 1)
        DC = ref.random_matrix(m, n, 12, 2)
        da, db, sr, sk = ref.tesseract_backward(DC, A, B, q, d, allow=allow)
        key = f"bwd_{q}{q}{d}"
        out.update({key + "_a": A, key + "_b": B, key + "_dc": DC, key + "_da": da,
                    key + "_db": db, key + "_sr": sr, key + "_sk": sk})
    # layer_run for every LayerOp at [2,2,2] (b=4, s=3, h=16, heads=4).
    b, s, h, nh = 4, 3, 16, 4
    x = ref.random_matrix(b * s, h, 13, 0)
    dy = ref.random_matrix(b * s, h, 13, 2)
    P = ref.random_block_params(h, 13, 100)
    out["layer_x"], out["layer_dy"] = x, dy
    for k_, v_ in P.items():
        out["layer_p_" + k_] = v_
    for op in oracle.LAYER_OPS:
        res = ref.layer_run(op, x, dy, P, b, s, nh, q=2, d=2)
        out[f"layer_{op}_y"], out[f"layer_{op}_dx"] = res["y"], res["dx"]
        out[f"layer_{op}_dbias"] = res["dbias"]
        out[f"layer_{op}_sk"] = res["stats_kind"]
        for k_, v_ in res["grads"].items():
            out[f"layer_{op}_g_{k_}"] = v_
    np.savez_compressed(os.path.join(HERE, "reference_small.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()


def traces():
    """Reference write_trace() text for NN/NT/TN (record_trace), small shapes."""
    import json
    ref = oracle.Reference()
    out = {}
    for q, d, allow in [(2, 1, False), (2, 2, False), (1, 2, True)]:
        m, n, r = 4 * q * d, 4 * q, 6 * q
        a = ref.random_matrix(m, n, 14, 0)
        for v, b in (("nn", ref.random_matrix(n, r, 14, 1)), ("nt", ref.random_matrix(r, n, 14, 1)),
                     ("tn", ref.random_matrix(m, r, 14, 1))):
            out[f"{v}_{q}{q}{d}"] = ref.tesseract_matmul_trace(a, b, q, d, v, allow=allow)
    with open(os.path.join(HERE, "reference_traces.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print("wrote", len(out), "traces")


if __name__ == "__main__" and "--traces" in sys.argv:
    traces()
