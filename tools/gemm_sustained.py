"""Sustained (power-capped) GEMM throughput: the tess tcgen05 GEMM vs cuBLAS
(torch.matmul), each run back to back for SECONDS with nvidia-smi sampling
SM clock and power during the run. Prints one JSON line per (shape, impl)."""
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2105_14500_b200 as tess  # noqa: E402

SECONDS = float(os.environ.get("SECONDS_PER_RUN", "4"))
SHAPES = [("sq8192_nn", 8192, 8192, 8192), ("ff1_nn", 8192, 49152, 12288)]


def sample(stop, out):
    p = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,power.draw",
                          "--format=csv,noheader,nounits", "-lms", "100"],
                         stdout=subprocess.PIPE, text=True)
    while not stop.is_set():
        line = p.stdout.readline()
        if line:
            out.append(line.strip())
    p.terminate()


def run(fn, flops):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    lines, stop = [], threading.Event()
    th = threading.Thread(target=sample, args=(stop, lines))
    th.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 0
    e0.record()
    t0 = time.time()
    while time.time() - t0 < SECONDS:
        for _ in range(10):
            fn()
        n += 10
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    ms = e0.elapsed_time(e1) / n
    clk = [float(x.split(",")[0]) for x in lines if x]
    pw = [float(x.split(",")[1]) for x in lines if x]
    return {"tflops": flops / ms / 1e9, "ms": ms, "iters": n,
            "sm_mhz_median": statistics.median(clk) if clk else None,
            "power_w_median": statistics.median(pw) if pw else None}


def main():
    dev = torch.device("cuda", 0)
    ctx = tess.init_local(tess.GridSpec(1, 1))[0]
    st = torch.cuda.current_stream().cuda_stream
    for name, M, N, K in SHAPES:
        a = torch.randn(M, K, device=dev, dtype=torch.bfloat16)
        b = torch.randn(K, N, device=dev, dtype=torch.bfloat16)
        c = torch.empty(M, N, device=dev, dtype=torch.bfloat16)

        def ours():
            ctx.matmul("nn", "bf16", a.data_ptr(), M, K, b.data_ptr(), K, N, c.data_ptr(),
                       c_dtype="bf16", stream=st)

        def ref():
            torch.matmul(a, b, out=c)
        for label, fn in (("cublas", ref), ("tess", ours), ("cublas", ref), ("tess", ours)):
            r = run(fn, 2.0 * M * N * K)
            r.update(shape=name, impl=label)
            print(json.dumps(r), flush=True)
            time.sleep(2)
        del a, b, c
        torch.cuda.empty_cache()
    ctx.close()


if __name__ == "__main__":
    main()
