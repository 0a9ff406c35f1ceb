"""Summarise an ncu `--metrics gpu__time_duration.sum --csv` launch list:
per-kernel total time, launches and share of the step. With a second path,
also writes {kernel: share of the step} keyed like tess.profile_kernels()
(bench.py's roofline.ncu_share_of_step).

  python tools/launch_summary.py launches.csv [profiles/ncu_launch_share.json]
"""
import collections
import csv
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_digest import our_name  # noqa: E402


def main(path, share_out=None):
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "nsecond")
        scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}.get(unit, 1e-6)
        name = r["Kernel Name"].split("(")[0]
        rows.append((name, v * scale))
    agg = collections.defaultdict(lambda: [0.0, 0])
    for n, ms in rows:
        agg[n][0] += ms
        agg[n][1] += 1
    tot = sum(a[0] for a in agg.values())
    print(f"total {tot:.3f} ms over {len(rows)} launches")
    for n, (ms, k) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        print(f"{ms:9.3f} ms {100 * ms / tot:5.1f}%  x{k:<4d} {n}")
    if share_out:
        share = collections.defaultdict(float)
        for n, (ms, _) in agg.items():
            share[our_name(n)] += ms / tot
        with open(share_out, "w") as f:
            json.dump(dict(sorted(share.items(), key=lambda kv: -kv[1])), f, indent=1)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
