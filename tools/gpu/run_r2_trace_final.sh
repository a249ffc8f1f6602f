# round 2 (late): the served bursty trace (f2) with the final kernels (persistent prefill attention,
# shape-agnostic prefill graphs): static / static_slo / adaptive
mkdir -p gpurun_out
timeout 2400 python tools/trace_bench.py --n-req 48 --qps 40 --max-iters 8000 --out gpurun_out/trace_cfg4_final.json > gpurun_out/trace_final.log 2>&1
tail -5 gpurun_out/trace_final.log
python - <<'PY'
import json
d=json.load(open('gpurun_out/trace_cfg4_final.json'))
for k, x in d['results'].items():
    print(k, {kk: (round(vv, 4) if isinstance(vv, float) else vv) for kk, vv in x.items() if not isinstance(vv, (list, dict))})
PY
