# A/B of the attention backward in the cfg4 bench step: two-pass (default) vs split
set -x
timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_headline.py -x -q -m gpu 2>&1 | tail -5
for rep in 1 2; do
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab_two_$rep.json 2> gpurun_out/ab_two_$rep.err
  TESS_ATTN_BWD_SPLIT=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab_split_$rep.json 2> gpurun_out/ab_split_$rep.err
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/ab_*.json')):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, 'ERR', e); continue
    pk=d['roofline'].get('per_kernel_ms_flops_launches_bytes',{})
    att={k:round(v[0],3) for k,v in pk.items() if 'attn' in k or '<128,1,1>' in k}
    print(f, round(d['value'],1), 'ms', round(d['ms_per_step'],2), 'mhz', d['clocks']['sm_mhz'], 'e2e', round(d['e2e']['value'],1), att)
PY
