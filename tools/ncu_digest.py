"""Digest an `ncu --set full` raw CSV of one step (tools/ncu_step.py) into
profiles/ncu_kernel_traffic.json: per kernel instantiation (named like
tess.profile_kernels(): gemm_bf16_2cta_kernel<am,bm,tile_n>, attn_*), the
mean DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum),
duration, tensor-pipe and L2 figures -- the `roofline.traffic` of bench.py.

  python tools/ncu_digest.py gpurun_out/step_full_raw.csv profiles/ncu_kernel_traffic.json
"""
import collections
import csv
import json
import re
import sys


def our_name(ncu_name):
    # <A_MN, B_MN, stages, halves[, pair MMA N]> -> tile width = halves * N
    m = re.search(r"gemm_bf16_2cta_kernel<(\w+), (\w+), (\d+), (\d+)(?:, (\d+))?(?:, (\d+))?>", ncu_name)
    if m:
        b = lambda v: "1" if v in ("true", "1") else "0"  # noqa: E731
        bnp = int(m[5]) if m[5] else 256
        return f"gemm_bf16_2cta_kernel<{b(m[1])},{b(m[2])},{bnp * int(m[4])}>"
    m = re.search(r"gemm_bf16_kernel<(\d+), (\w+), (\w+)>", ncu_name)
    if m:
        b = lambda v: "1" if v in ("true", "1") else "0"  # noqa: E731
        return f"gemm_bf16_kernel<{m[1]},{b(m[2])},{b(m[3])}>"
    m = re.search(r"(attn_\w+_kernel<\d+>)", ncu_name)
    if m:
        return m[1]
    m = re.search(r"(\w+_kernel)\b", ncu_name)  # memory-bound kernels: base name
    return m[1] if m else ncu_name.split("(")[0].replace("void ", "")


KEEP = {
    "gpu__time_duration.sum": "ms",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    # tcgen05 (UTC) bf16 MMA ops as % of the tensor peak at the kernel's clock
    "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed":
        "tensor_bf16_pct_of_peak",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_active_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "sm__cycles_elapsed.avg.per_second": "sm_hz",
}


def main(src, dst):
    with open(src) as f:
        rows = list(csv.reader(f))
    hdr = rows[0]
    units = rows[1] if len(rows) > 1 else []
    idx = {h: i for i, h in enumerate(hdr)}
    name_col = idx.get("Kernel Name")
    agg = collections.defaultdict(lambda: collections.defaultdict(list))
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        n = our_name(r[name_col])
        for metric, key in KEEP.items():
            if metric not in idx:
                continue
            try:
                v = float(r[idx[metric]].replace(",", ""))
            except ValueError:
                continue
            u = units[idx[metric]] if units else ""
            if metric == "gpu__time_duration.sum":
                v *= {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "ms": 1.0,
                      "us": 1e-3, "ns": 1e-6}.get(u, 1e-6)
            if metric.endswith("per_second"):
                v *= {"hz": 1, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9}.get(u, 1)
            if metric.startswith("dram__bytes"):
                v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)
            agg[n][key].append(v)
    out = {}
    for n, d in agg.items():
        e = {k: sum(v) / len(v) for k, v in d.items()}
        e["launches"] = len(d.get("ms", []))
        if "dram_read" in e and "dram_write" in e:
            e["dram_bytes_per_launch"] = e["dram_read"] + e["dram_write"]
        out[n] = e
    with open(dst, "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    for n, e in sorted(out.items(), key=lambda kv: -kv[1].get("ms", 0) * kv[1]["launches"]):
        print(f"{n:40s} x{e['launches']:<3d} ms {e.get('ms', 0):7.3f} dram/launch "
              f"{e.get('dram_bytes_per_launch', 0) / 1e9:6.2f} GB tensor(bf16 ops % of peak) "
              f"{e.get('tensor_bf16_pct_of_peak', float('nan')):5.1f}% L2hit {e.get('l2_hit_pct', 0):5.1f}%"
              f" {e.get('sm_hz', 0) / 1e6:5.0f} MHz")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
