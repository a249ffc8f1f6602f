mkdir -p gpurun_out
[ -n "$SKIPTEST" ] || DUET_DECODE=p2w2x6 timeout 600 python -m pytest tests -m gpu -x -q -k "tiny or llama or invariant" 2>&1 | tail -2
for v in ${VARIANTS:-cp4x3x2 p2w2x6}; do
  DUET_DECODE=$v timeout 300 python tools/partition_bench.py --only decode --out gpurun_out/dec_$v.json > /dev/null 2>&1
  python - "$v" <<'PY'
import json,sys
v=sys.argv[1]
d=json.load(open(f'gpurun_out/dec_{v}.json'))
print(v.ljust(8), ' '.join(f"{r['sms']}:{r['kernels']['decode_attn']['s_per_launch']*1e6:.0f}us/{r['t_meas_ms']:.3f}ms" for r in d['rows'] if r['sms'] in (8,16,24,32,48,148)))
PY
done
