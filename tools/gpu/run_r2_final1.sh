# round 2: sanitizers, full GPU suite, smoke, cfg3 bench (default) + cfg2 line
mkdir -p gpurun_out
bash tools/gpu/run_r2_sanitize.sh
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/tests_final1.log; cat gpurun_out/tests_final1.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 1800 python bench.py > gpurun_out/bench_cfg3_f.json 2> gpurun_out/bench_cfg3_f.log
grep -E "split:|timed:" gpurun_out/bench_cfg3_f.log
python - <<'PY'
import json
d=json.load(open('gpurun_out/bench_cfg3_f.json'))
print(d['value'], d['ms_per_step'], d['config']['s_d'], d['config']['k'], d['clocks']['sm_mhz'], d['steps'], d['warmup'])
c=d['comparison']
for k in ('aggregated_chunked_at_slo','partitioned_optimizer','partitioned_boundary_aware'):
    v=c.get(k)
    if v: print(k, round(v['tok_s']), round(v['window_ms'],1), v['k'], round(v['t_decode_ms']/v['k'],1), round(v.get('tbt_max_ms',0),1), v.get('sm_mhz'))
print(json.dumps(d['roofline'])[:300])
PY
