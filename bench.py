#!/usr/bin/env python3
"""Benchmark: Tesseract Transformer-layer fwd+bwd on B200 (BASELINE.json).

Workload (BASELINE.json configs[3], weak scaling): one pre-norm Transformer
block (LN -> QKV -> attention (no mask) -> proj -> +res -> LN -> FF1+GeLU ->
FF2 -> +res), forward + backward with weight/LN gradients, h=12288, 96 heads,
seq 2048, batch 4 per GPU-equivalent (b = 4 * p), bf16 storage with fp32
accumulation, on the [q,q,d] grid for N GPUs:
    N=1 [1,1,1]   N=2 [1,1,2]   N=4 [2,2,1]   N=8 [2,2,2]
One process per GPU (torchrun for N>1; started without torchrun and with
--gpus N > 1, bench.py re-launches itself under torch.distributed.run), NCCL
row/column/depth communicators inside libtess; torch.distributed (gloo) only
for the unique-id exchange, barriers and the max-over-ranks timing
reduction. Synthetic weights are seeded per TesseractB block (i, j), so the
depth replicas of a weight block are identical; `--dry-run` stops after the
rendezvous and prints every rank's (rank, device, coordinate).

Prints ONE JSON line on rank 0 (see the contract in the task statement).
`--impl reference` times the reference's own CPU implementation
(oracle/_ref, the unmodified tesseract-sim) on a bounded sample instead.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2105_14500_b200.launch import GRIDS, grid_for, rank_env, seeds, spawn  # noqa: E402

METRIC = "Transformer-layer fwd+bwd TFLOP/s at [2,2,2] on 8×B200; step ms; exposed comm %"
HIDDEN, HEADS, SEQ, B_PER_GPU = 12288, 96, 2048, 4
# CPU sample for the reference / cpu_baseline legs (bounded CPU work)
SAMPLE = dict(batch=4, seq=128, hidden=512, heads=8)


def arm_config(gpus, grid_str=None):
    """The `config` both arms report: BASELINE configs[3] at this GPU count."""
    q, d, _ = GRIDS.get(gpus, (1, 1, True))
    p = d * q * q
    batch = B_PER_GPU * p
    return {"workload": "cfg4: Tesseract Transformer block fwd+bwd (attention, no mask, + "
                        "MLP + distributed LayerNorm), weak scaling b=4*p",
            "grid": grid_str or f"[{q},{q},{d}]", "global_batch": batch, "seq_len": SEQ,
            "hidden": HIDDEN, "heads": HEADS, "rows_per_rank": batch * SEQ // (d * q),
            "parallelism": f"tesseract[{q},{q},{d}]",
            "l2": "inputs larger than L2 (per-GPU weights+activations >> 126 MB)"}


# BASELINE configs[4]: 24-layer hidden-4096 stack, strong scaling (SURVEY 8d
# proposal s=2048, b=16, 32 heads), Tesseract vs 1-D vs SUMMA
CFG5 = dict(layers=24, hidden=4096, heads=32, seq=2048, batch=16)


def grid_for_scheme(gpus, scheme):
    """(q, d, allow) of a config-5 scheme on `gpus` ranks: Tesseract as the
    cfg4 ladder, SUMMA [q,q,1] (q*q == gpus), the 1-D scheme a [1,1,gpus] line."""
    if scheme == "tesseract":
        return grid_for(gpus)
    if scheme == "summa":
        q = int(round(gpus ** 0.5))
        if q * q != gpus:
            raise SystemExit("SUMMA needs a square GPU count (1 or 4)")
        return q, 1, False
    if scheme == "megatron":
        return 1, gpus, True
    raise SystemExit(f"unknown scheme {scheme}")


def cfg5_config(args, grid_str):
    return {"workload": f"cfg5: {args.layers}-layer Transformer stack fwd+bwd (pre-norm blocks, "
                        f"attention no mask + MLP + LayerNorm), strong scaling, scheme "
                        f"{args.scheme}",
            "grid": grid_str, "scheme": args.scheme, "layers": args.layers,
            "global_batch": args.batch, "seq_len": args.seq, "hidden": args.hidden,
            "heads": args.heads, "parallelism": f"{args.scheme}{grid_str}",
            "l2": "inputs larger than L2 (per-GPU weights+activations >> 126 MB)"}


def layer_flops(batch, seq, hidden):
    """Algorithmic flops of one block fwd+bwd (2*m*n*k of GEMMs + attention
    contractions): 72*T*h^2 + 12*T*s*h, T = batch*seq."""
    T = batch * seq
    return 72.0 * T * hidden * hidden + 12.0 * T * seq * hidden


def read_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d.get("bf16_tflops_sustained", 1434.2), "measured", d.get("hbm_gbs")
    return 1400.0, "fallback", 6650.0


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.lines = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def mark(self, which):
        """Host time bounds of the timed region (samples outside are dropped)."""
        setattr(self, which, time.time())

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        t0, t1 = getattr(self, "t0", None), getattr(self, "t1", None)
        for ts, ln in self.lines:
            if t0 is not None and t1 is not None and not (t0 <= ts <= t1 + 0.15):
                continue
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------- CPU legs
def cpu_sample_run(reps_min_s=10.0, reps_max_s=30.0, max_reps=None):
    """Times the reference CPU implementation of layer_run(Block) on the
    bounded SAMPLE; returns (tflops, seconds_per_call, kind, cores, desc)."""
    import numpy as np
    ncpu = os.cpu_count() or 1
    os.environ.setdefault("OMP_NUM_THREADS", str(ncpu))
    import oracle
    b, s, h, nh = SAMPLE["batch"], SAMPLE["seq"], SAMPLE["hidden"], SAMPLE["heads"]
    orc = oracle.Oracle()
    x = orc.random_matrix(b * s, h, 42, 0)
    dy = orc.random_matrix(b * s, h, 42, 2)
    P = orc.random_block_params(h, 42, 100)
    if oracle.Reference.available():
        ref = oracle.Reference()
        kind, cores = "reference", int(os.environ.get("OMP_NUM_THREADS", ncpu))
        call = lambda: ref.layer_run("block", x, dy, P, b, s, nh, q=1, d=1)  # noqa: E731
    else:
        kind, cores = "port", 1
        call = lambda: orc.layer_run("block", x, dy, P, b, s, nh)  # noqa: E731
    times = []
    t_all = time.perf_counter()
    while True:
        t0 = time.perf_counter()
        call()
        times.append(time.perf_counter() - t0)
        el = time.perf_counter() - t_all
        if max_reps is not None:
            if len(times) >= max_reps:
                break
            continue
        if el >= reps_min_s or el + times[-1] > reps_max_s:
            break
    per = sum(times) / len(times)
    fl = layer_flops(b, s, h)
    desc = (f"layer_run(Block) fwd+bwd b={b} s={s} h={h} heads={nh} grid [1,1,1], "
            f"{len(times)} calls, fp64")
    return fl / per / 1e12, per, kind, cores, desc, np


def cpu_legs():
    """config 1 tesseract_matmul / tesseract_backward_dense
    at full size and the Block sample, best of 3, each with OMP_NUM_THREADS =
    nproc and = 1 (each its own process: OpenMP reads it once)."""
    out = {}
    for omp in (os.cpu_count() or 1, 1):
        env = dict(os.environ, OMP_NUM_THREADS=str(omp))
        try:
            r = subprocess.run([sys.executable, "-m", "oracle.cpu_legs"], cwd=ROOT, env=env,
                               capture_output=True, text=True, timeout=240)
            out[f"omp{omp}"] = json.loads(r.stdout.strip().splitlines()[-1])
        except (subprocess.SubprocessError, ValueError, IndexError) as e:
            out[f"omp{omp}"] = {"error": str(e)[:200]}
    return out


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    fl = layer_flops(SAMPLE["batch"], SAMPLE["seq"], SAMPLE["hidden"])
    # warmup + timed steps, one sample call per step
    cpu_sample_run(max_reps=max(args.warmup, 1), reps_min_s=0, reps_max_s=1e9)
    tf, per, kind, cores, desc, _ = cpu_sample_run(max_reps=args.steps, reps_min_s=0,
                                                   reps_max_s=1e9)
    line = {"metric": METRIC, "value": tf, "unit": "TFLOP/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": per * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            # same workload as the GPU arm; each step runs a bounded sample of it
            # (flop-normalised, see cpu_baseline.sample)
            "config": {**arm_config(args.gpus), "reference_sample": dict(SAMPLE)},
            "cpu_baseline": {"value": tf, "unit": "TFLOP/s", "cores": cores, "kind": kind,
                             "sample": desc},
            "e2e": {"value": tf, "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------- GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="tess", choices=["tess", "reference"])
    ap.add_argument("--batch-per-gpu", type=int, default=B_PER_GPU)
    ap.add_argument("--hidden", type=int, default=HIDDEN)
    ap.add_argument("--heads", type=int, default=HEADS)
    ap.add_argument("--seq", type=int, default=SEQ)
    ap.add_argument("--workload", default="cfg4", choices=["cfg4", "cfg5"],
                    help="cfg4: one block, weak scaling (default, the headline); cfg5: the "
                         "24-layer h=4096 stack under --scheme, strong scaling")
    ap.add_argument("--scheme", default="tesseract", choices=["tesseract", "summa", "megatron"])
    ap.add_argument("--layers", type=int, default=None)
    ap.add_argument("--batch", type=int, default=None, help="cfg5 global batch")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--dry-run", action="store_true",
                    help="stop after the rendezvous; rank 0 prints each rank's placement")
    args = ap.parse_args()
    if args.workload == "cfg5":
        for k, v in CFG5.items():
            if getattr(args, k) is None or (k in ("hidden", "heads", "seq") and
                                            getattr(args, k) == ap.get_default(k)):
                setattr(args, k, v)
        args.no_cpu_baseline = True
    else:
        args.layers = 1

    rank, local_rank, world = rank_env()
    if world == 1 and args.gpus > 1 and args.impl == "tess":
        # started without torchrun: one process per GPU, this one only launches
        grid_for(args.gpus)
        raise SystemExit(spawn(os.path.abspath(__file__), sys.argv[1:], args.gpus))
    if world > 1:
        args.gpus = world
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")

    if args.dry_run:
        import paper_2105_14500_b200 as tess
        q, d, allow = grid_for_scheme(args.gpus,
                                      args.scheme if args.workload == "cfg5" else "tesseract")
        grid = tess.GridSpec(q, d, allow)
        c = grid.coord_of(rank)
        me = {"rank": rank, "local_rank": local_rank, "device": local_rank,
              "coord": [c.i, c.j, c.k], "grid": grid.to_string(), "seeds": seeds(grid, rank)}
        allr = [None] * world
        if dist:
            dist.all_gather_object(allr, me)
        else:
            allr = [me]
        if rank == 0:
            print(json.dumps({"dry_run": True, "world": world, "ranks": allr}), flush=True)
        if dist:
            dist.barrier()
            dist.destroy_process_group()
        return

    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        if dist:
            dist.barrier()
        return

    import torch
    import paper_2105_14500_b200 as tess

    cfg5 = args.workload == "cfg5"
    q, d, allow = grid_for_scheme(args.gpus, args.scheme if cfg5 else "tesseract")
    grid = tess.GridSpec(q, d, allow)
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)

    if world > 1:
        obj = [tess.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ctx = tess.init_nccl(grid, rank, local_rank, obj[0])
    else:
        ctx = tess.init_local(grid)[0]

    p = grid.size()
    h, nh, s = args.hidden, args.heads, args.seq
    L = args.layers
    mg = args.scheme == "megatron"
    if mg:
        ctx.set_megatron(True)
    # cfg4 weak scaling: b = 4 per GPU; cfg5 strong scaling: b fixed for the job
    batch = args.batch if cfg5 else args.batch_per_gpu * p
    dims = tess.LayerDims(batch, s, h, nh)
    # this rank's activation block: TesseractA [T/(d q), h/q]; 1-D: all of [T, h]
    rows = batch * s if mg else batch * s // (d * q)
    hin = h if mg else h // q
    bf = torch.bfloat16
    sd = seeds(grid, rank)
    if mg:  # 1-D: activations replicated, weight shards differ per rank
        sd = {"activation": 1234 + 1000, "weight": 1234 + 2000 + rank, "ln": 1234 + 3000}
    gens = {}
    for fam, seed in sd.items():
        gens[fam] = torch.Generator(device=dev)
        gens[fam].manual_seed(seed)

    def rnd(shape, scale, fam, dtype=bf):
        return (torch.rand(shape, device=dev, generator=gens[fam]) * 2 - 1).mul_(scale).to(dtype)

    # synthetic inputs of the named shapes; random-init weights: TesseractB
    # blocks seeded by (i, j) (identical depth replicas), LN by j. 1-D scheme:
    # W_qkv / W_ff1 column shards, W_proj / W_ff2 row shards, full LN vectors.
    ws = 1.0 / (h ** 0.5)
    if mg:
        hp = h // p
        wshape = {"w_qkv": (h, 3 * hp), "w_proj": (hp, h), "w_ff1": (h, 4 * hp),
                  "w_ff2": (4 * hp, h)}
    else:
        hq = h // q
        wshape = {"w_qkv": (hq, 3 * hq), "w_proj": (hq, hq), "w_ff1": (hq, 4 * hq),
                  "w_ff2": (4 * hq, hq)}
    keep = []
    shards, gradl = [], []
    for _ in range(L):
        W = {k: rnd(v, ws, "weight") for k, v in wshape.items()}
        LN = {k: (1 if k.endswith("gain") else 0) + rnd((hin,), 0.1, "ln", torch.float32)
              for k in ("ln1_gain", "ln1_bias", "ln2_gain", "ln2_bias")}
        G = {k: torch.empty(v.shape, dtype=torch.float32, device=dev)
             for k, v in {**W, **LN}.items()}
        keep.append((W, LN, G))
        shards.append(tess.BlockShardC(
            *[W[k].data_ptr() for k in ("w_qkv", "w_proj", "w_ff1", "w_ff2")],
            *[LN[k].data_ptr() for k in ("ln1_gain", "ln1_bias", "ln2_gain", "ln2_bias")], 1e-5))
        gradl.append(tess.BlockGradsC(*[G[k].data_ptr() for k in tess.PARAM_NAMES]))
    shard, grads = shards[0], gradl[0]
    x = rnd((rows, hin), 1.0, "activation")
    dy = rnd((rows, hin), 1.0, "activation")
    y = torch.empty_like(x)
    dx = torch.empty_like(x)
    stream = torch.cuda.current_stream(dev)
    sh = stream.cuda_stream

    if cfg5:
        def step(xp, yp, dyp, dxp):
            ctx.stack_step("bf16", dims, shards, xp, dyp, yp, dxp, gradl, stream=sh)
        step_api = step
    else:
        def step(xp, yp, dyp, dxp):
            ctx.layer_forward("block", "bf16", dims, shard, xp, yp, stream=sh)
            ctx.layer_backward("block", "bf16", dims, shard, dyp, dxp, grads, accumulate=False,
                               stream=sh)

        def step_api(xp, yp, dyp, dxp):
            # the user-facing call for a training step of the layer (rank-level
            # layer_run: forward + backward with x and dy given together)
            ctx.layer_step("block", "bf16", dims, shard, xp, dyp, yp, dxp, grads,
                           accumulate=False, stream=sh)

    def barrier():
        torch.cuda.synchronize(dev)
        if dist:
            dist.barrier()

    def max_over_ranks(v):
        if not dist:
            return v
        t = torch.tensor([v], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # the sampler starts before the warm-up (nvidia-smi needs ~0.5 s to come
    # up) and keeps only the samples taken inside the timed region
    clocks = ClockSampler(local_rank)
    clocks.start()
    for _ in range(args.warmup):
        step(x.data_ptr(), y.data_ptr(), dy.data_ptr(), dx.data_ptr())
    barrier()
    launches0 = tess.kernel_launches()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # The timed region: K steps; every tensor-core launch (GEMMs, fused
    # attention) and every memory-bound launch (LayerNorm, attention delta,
    # ...) bracketed by CUDA events on its own stream, so the roofline's
    # per-kernel times come from this very region.
    tess.profile_enable(True)
    barrier()
    clocks.mark("t0")
    e0.record(stream)
    for _ in range(args.steps):
        step(x.data_ptr(), y.data_ptr(), dy.data_ptr(), dx.data_ptr())
    e1.record(stream)
    barrier()
    clocks.mark("t1")
    clk = clocks.stop()
    launches = tess.kernel_launches() - launches0
    ms_local = e0.elapsed_time(e1) / args.steps
    ms = max_over_ranks(ms_local)
    flops = L * layer_flops(batch, s, h)
    value = flops / (ms * 1e-3) / 1e12
    gemm_ms, gemm_flops, gemm_n = tess.profile_read()
    per_kernel = tess.profile_kernels()
    tess.profile_enable(False)
    # the same K steps without the per-launch events (their cost, reported)
    barrier()
    e0.record(stream)
    for _ in range(args.steps):
        step(x.data_ptr(), y.data_ptr(), dy.data_ptr(), dx.data_ptr())
    e1.record(stream)
    barrier()
    ms_unprof = max_over_ranks(e0.elapsed_time(e1) / args.steps)

    # exposed communication: the same step with every collective
    # metered but moving no data; exposed = (t - t_noop) / t, max over ranks.
    # A one-rank grid has no collectives at all: exposed is 0 by construction.
    if p == 1:
        ms_noop, exposed = ms, 0.0
    else:
        ctx.set_comm_noop(True)
        for _ in range(2):
            step(x.data_ptr(), y.data_ptr(), dy.data_ptr(), dx.data_ptr())
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            step(x.data_ptr(), y.data_ptr(), dy.data_ptr(), dx.data_ptr())
        e1.record(stream)
        barrier()
        ctx.set_comm_noop(False)
        ms_noop = max_over_ranks(e0.elapsed_time(e1) / args.steps)
        exposed = max(0.0, (ms - ms_noop) / ms) if ms else None

    # per-launch averages over the K timed steps (rank 0's own kernels)
    ms_prof = ms_local
    K = float(args.steps)
    peak, peak_src, hbm_peak = read_peaks()
    tensor = {k: v for k, v in per_kernel.items() if v[1] > 0}
    memory = {k: v for k, v in per_kernel.items() if v[1] == 0}
    # dominant kernel = the tensor-core instantiation with the most device
    # time; achieved = its algorithmic flops per launch / its mean launch time
    top, (top_ms, top_flops, top_n, _) = max(tensor.items(), key=lambda kv: kv[1][0])
    achieved = top_flops / (top_ms * 1e-3) / 1e12 if top_ms > 0 else None
    # the same figure from the committed ncu launch list of one step (its
    # SHARE of the step, cold-cache and serialised) x this run's step time
    share = None
    sp = os.path.join(ROOT, "profiles", "ncu_launch_share.json")
    # the committed ncu captures are of the cfg4 step: not quoted for cfg5
    if os.path.exists(sp) and not cfg5:
        with open(sp) as f:
            share = json.load(f).get(top)
    achieved_ncu = (top_flops / top_n) / (share * ms / (top_n / K) * 1e-3) / 1e12 \
        if share else None
    # DRAM bytes per launch of that kernel from the committed `ncu --set full`
    # capture of one step (tools/ncu_step.py -> tools/ncu_digest.py)
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_kernel_traffic.json")
    if os.path.exists(tp) and not cfg5:
        with open(tp) as f:
            traffic = json.load(f).get(top, {}).get("dram_bytes_per_launch")
    burst = None
    pk = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(pk):
        with open(pk) as f:
            burst = json.load(f).get("bf16_tflops")
    # step accounting: device time of every profiled launch vs the step
    prof_sum = sum(v[0] for v in per_kernel.values()) / K
    hbm = {k: {"ms_per_launch": v[0] / v[2], "launches_per_step": v[2] / K,
               "bytes_per_launch": v[3] / v[2],
               "gbs": v[3] / (v[0] * 1e-3) / 1e9 if v[0] > 0 else None,
               "frac_of_hbm_peak": (v[3] / (v[0] * 1e-3) / 1e9) / hbm_peak
               if v[0] > 0 and hbm_peak else None}
           for k, v in sorted(memory.items())}

    # end to end through the C-ABI with host (pinned) buffers, copies inside
    e2e = None
    if not args.no_e2e:
        xh = x.cpu().pin_memory()
        dyh = dy.cpu().pin_memory()
        yh = torch.empty_like(xh).pin_memory()
        dxh = torch.empty_like(xh).pin_memory()
        for _ in range(max(1, args.warmup)):
            step_api(xh.data_ptr(), yh.data_ptr(), dyh.data_ptr(), dxh.data_ptr())
        ctx.stream_join(sh)
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            step_api(xh.data_ptr(), yh.data_ptr(), dyh.data_ptr(), dxh.data_ptr())
        ctx.stream_join(sh)  # the last step's host copies complete inside the timed region
        e1.record(stream)
        barrier()
        ms_e2e = max_over_ranks(e0.elapsed_time(e1) / args.steps)
        nbytes = xh.numel() * xh.element_size()
        e2e = {"value": flops / (ms_e2e * 1e-3) / 1e12, "unit": "TFLOP/s",
               "ms_per_step": ms_e2e, "h2d_bytes_per_step": 2 * nbytes * p,
               "d2h_bytes_per_step": 2 * nbytes * p}

    cpu = None
    if rank == 0 and args.gpus == 1 and not args.no_cpu_baseline:
        tf, per, kind, cores, desc, _ = cpu_sample_run()
        cpu = {"value": tf, "unit": "TFLOP/s", "cores": cores, "kind": kind, "sample": desc,
               "seconds_per_call": per, "omp_num_threads": cores,
               "sample_scale": "cfg4 tokens x1/16 (T=512 vs 8192), hidden x1/24 (512 vs "
                               "12288), heads 8 vs 96; flop-normalised",
               "legs": cpu_legs()}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong" if cfg5 else "weak",
            "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (random inputs and random-init weights of the named shapes)",
            "config": cfg5_config(args, grid.to_string()) if cfg5
            else arm_config(args.gpus, grid.to_string()),
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak,
                         "peak_source": f"{peak_src} bf16_tflops_sustained", "unit": "TFLOP/s",
                         "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                         "kernel": top, "kernel_launches_per_step": top_n / K,
                         "kernel_flops_per_launch": top_flops / top_n,
                         "kernel_ms_per_launch": top_ms / top_n,
                         "kernel_share_of_step": top_ms / K / ms_prof,
                         "timing": "CUDA events around each launch inside the timed region",
                         "ms_per_step_without_launch_events": ms_unprof,
                         "ncu_share_of_step": share,
                         "achieved_from_ncu_share": achieved_ncu,
                         "frac_from_ncu_share": achieved_ncu / peak if achieved_ncu else None,
                         "frac_of_burst_peak": (achieved / burst) if achieved and burst else None,
                         # every tensor-core launch of the step (GEMMs + fused attention)
                         "tensor_kernels_tflops": gemm_flops / (gemm_ms * 1e-3) / 1e12,
                         "tensor_kernels_ms_per_step": gemm_ms / K,
                         "tensor_kernels_launches_per_step": gemm_n / K,
                         "tensor_kernels_share_of_step": gemm_ms / K / ms_prof,
                         "profiled_kernels_ms_per_step": prof_sum,
                         "unprofiled_ms_per_step": ms_prof - prof_sum,
                         "per_kernel_ms_flops_launches_bytes":
                             {k: [v[0] / K, v[1] / K, v[2] / K, v[3] / K]
                              for k, v in per_kernel.items()},
                         "hbm_kernels": hbm, "hbm_peak_gbs": hbm_peak},
            "exposed_comm_pct": 100.0 * exposed if exposed is not None else None,
            "ms_per_step_without_comm": ms_noop,
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
