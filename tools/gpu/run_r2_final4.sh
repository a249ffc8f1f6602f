# round 2 (late): full GPU suite with f3, smoke, default cfg3 bench, cfg2 line
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/tests_final4.log; cat gpurun_out/tests_final4.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1800 python bench.py > gpurun_out/bench_cfg3_h.json 2> gpurun_out/bench_cfg3_h.log
python - <<'PY'
import json
d=json.load(open('gpurun_out/bench_cfg3_h.json'))
print(d['value'], d['ms_per_step'], d['config']['s_d'], d['config']['k'], d['clocks']['sm_mhz'], d['roofline']['frac'])
c=d['comparison']
for k in ('aggregated','aggregated_chunked_at_slo','partitioned_optimizer','partitioned_boundary_aware'):
    v=c.get(k)
    if v: print(k, round(v['tok_s']), round(v['window_ms'],1), v['k'], round(v.get('tbt_median_ms',0),1), round(v.get('tbt_max_ms',0),1), v.get('sm_mhz'))
print(json.dumps(d['predictor']['per_side']))
PY
timeout 900 python bench.py --config cfg2 --steps 50 --warmup 5 > gpurun_out/bench_cfg2_h.json 2> gpurun_out/bench_cfg2_h.log
python3 -c "import json; d=json.load(open('gpurun_out/bench_cfg2_h.json')); print('cfg2', d['value'], d['ms_per_step'], d['roofline']['frac'])"
