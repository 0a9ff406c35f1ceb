"""TEST / BASELINE INFRASTRUCTURE ONLY (bench.py's cpu_baseline leg runs it
in a subprocess): times the unmodified reference (oracle/_ref/libtsim_ref.so,
else the plain-C restatement) per BASELINE.md section 3 and prints one JSON
object. OMP_NUM_THREADS is read once by OpenMP at load, so each thread
setting is its own process:

    OMP_NUM_THREADS=1 python -m oracle.cpu_legs

Legs (one warm-up, best of 3; inputs from Rng::stream(42, id), rng.hpp):
  * config 1: tesseract_matmul NN, A, B 1024 x 1024, grid [2,2,2]
    (algorithms.cpp:131-186), full size;
  * config 1 backward: tesseract_backward_dense at the same size
    (algorithms.cpp:234-242), full size;
  * layer_run(Block) on the bench's bounded sample (layers.cpp:604-692),
    grid [1,1,1]: b=4, s=128, h=512, 8 heads = cfg4 scaled by 1/16 in tokens
    and 1/24 in hidden (flop-normalised to TFLOP/s).
"""
import json
import os
import platform
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402

SAMPLE = dict(batch=4, seq=128, hidden=512, heads=8)


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def best_of(call, reps=3):
    call()  # warm-up
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        call()
        ts.append(time.perf_counter() - t0)
    return min(ts)


def block_flops(b, s, h):
    T = b * s
    return 72.0 * T * h * h + 12.0 * T * s * h


def main():
    ref_ok = oracle.Reference.available()
    R = oracle.Reference() if ref_ok else oracle.Oracle()
    orc = oracle.Oracle()
    legs = {}
    a = orc.random_matrix(1024, 1024, 42, 0)
    b = orc.random_matrix(1024, 1024, 42, 1)
    dc = orc.random_matrix(1024, 1024, 42, 2)
    if ref_ok:
        t = best_of(lambda: R.tesseract_matmul(a, b, 2, 2, "nn"))
        legs["cfg1_tesseract_matmul_nn_1024_[2,2,2]"] = {"s": t, "gflops": 2 * 1024 ** 3 / t / 1e9}
        t = best_of(lambda: R.tesseract_backward(dc, a, b, 2, 2))
        legs["cfg1_tesseract_backward_dense_1024_[2,2,2]"] = {
            "s": t, "gflops": 4 * 1024 ** 3 / t / 1e9}
    bb, s, h, nh = SAMPLE["batch"], SAMPLE["seq"], SAMPLE["hidden"], SAMPLE["heads"]
    x = orc.random_matrix(bb * s, h, 42, 0)
    dy = orc.random_matrix(bb * s, h, 42, 2)
    P = orc.random_block_params(h, 42, 100)
    if ref_ok:
        call = lambda: R.layer_run("block", x, dy, P, bb, s, nh, q=1, d=1)  # noqa: E731
    else:
        call = lambda: R.layer_run("block", x, dy, P, bb, s, nh)  # noqa: E731
    t = best_of(call, reps=2)
    legs["cfg4_sample_layer_run_block_[1,1,1]"] = {
        "s": t, "tflops": block_flops(bb, s, h) / t / 1e12,
        "scale": "b=4 s=128 h=512 heads=8: cfg4 tokens x1/16, hidden x1/24"}
    print(json.dumps({"kind": "reference" if ref_ok else "port", "cpu_model": cpu_model(),
                      "nproc": os.cpu_count(),
                      "omp_num_threads": int(os.environ.get("OMP_NUM_THREADS", "0") or 0),
                      "legs": legs}))


if __name__ == "__main__":
    main()
