# round 2 (final): full GPU suite, smoke, default cfg3 bench after the last refactors
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -8 > gpurun_out/tests_final6.log; cat gpurun_out/tests_final6.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1800 python bench.py > gpurun_out/bench_cfg3_final.json 2> gpurun_out/bench_cfg3_final.log
python - <<'PY'
import json
d=json.load(open('gpurun_out/bench_cfg3_final.json'))
print(round(d['value']), d['ms_per_step'], d['config']['s_d'], d['config']['k'], d['clocks']['sm_mhz'], d['roofline']['kernel'], round(d['roofline']['frac'],3), d['roofline'].get('partition',{}).get('frac'))
c=d['comparison']
for k in ('aggregated','aggregated_chunked_at_slo','partitioned_optimizer','partitioned_boundary_aware'):
    v=c.get(k)
    if v: print(' ', k, round(v['tok_s']), round(v['window_ms'],1), v['k'], v.get('s_d'), round(v.get('tbt_median_ms',0),1), round(v.get('tbt_max_ms',0),1), v.get('sm_mhz'))
print(' ', json.dumps(d['predictor']['per_side']))
print(' e2e', d['e2e']['value'], 'cpu', d['cpu_baseline']['value'])
PY
