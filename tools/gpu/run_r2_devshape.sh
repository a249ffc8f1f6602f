# round 2 (late): shape-agnostic prefill graphs (device-side row counts) — parity, then the cfg3 line
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity_deep.py -x -q 2>&1 | tail -4
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_f3.py -x -q -k "spatial or split or graph or trace or fused or mini" 2>&1 | tail -3
timeout 1800 python bench.py > gpurun_out/bench_cfg3_k.json 2> gpurun_out/bench_cfg3_k.log
python - <<'PY'
import json
d=json.load(open('gpurun_out/bench_cfg3_k.json'))
print(round(d['value']), d['ms_per_step'], d['config']['s_d'], d['config']['k'], d['clocks']['sm_mhz'])
c=d['comparison']
for k in ('aggregated_chunked_at_slo','partitioned_optimizer'):
    v=c.get(k)
    if v: print(' ', k, round(v['tok_s']), round(v['window_ms'],1), v['k'], v.get('s_d'), round(v.get('t_decode_ms',0),1), round(v.get('t_prefill_ms',0),1), v.get('prefill_graph'), v.get('sm_mhz'))
print(' ', json.dumps(d['predictor']['per_side']))
PY
