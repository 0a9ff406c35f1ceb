for r in 1 2 3; do timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b3_$r.json 2>/dev/null; done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/b3_*.json')):
    d=json.loads(open(f).read().strip().splitlines()[-1]); pk=d['roofline']['per_kernel_ms_flops_launches_bytes']
    print(f, round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'mhz', d['clocks']['sm_mhz'], {k:round(v[0],3) for k,v in pk.items() if 'attn' in k or 'ln_' in k})
PY
