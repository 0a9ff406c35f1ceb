# same-box A/B of two libtess builds in the cfg4 bench step (tools/libvar/libtess_{A,B}.so)
cp paper_2105_14500_b200/libtess.so /tmp/libtess_cur.so
for rep in 1 2; do
  for v in A B; do
    cp tools/libvar/libtess_$v.so paper_2105_14500_b200/libtess.so
    timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab_$v.$rep.json 2>/dev/null
  done
done
cp /tmp/libtess_cur.so paper_2105_14500_b200/libtess.so
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/ab_[AB].*.json')):
    try: d=json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e: print(f,'ERR',e); continue
    pk=d['roofline']['per_kernel_ms_flops_launches_bytes']
    print(f, round(d['value'],1), 'ms', round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value'],1), 'mhz', d['clocks']['sm_mhz'], {k:round(v[0],3) for k,v in pk.items() if 'attn' in k})
PY
