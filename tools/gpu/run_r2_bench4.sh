# round 2: device-timer test + cfg3 bench (decode attention timed inside the decode graph)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_profile.py -m gpu -x -q 2>&1 | tail -3
timeout 1800 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_cfg3_d.json 2> gpurun_out/bench_cfg3_d.log
grep -E "split:|timed:" gpurun_out/bench_cfg3_d.log
python - <<'PY'
import json
d=json.load(open('gpurun_out/bench_cfg3_d.json'))
print(d['value'], d['ms_per_step'], d['config']['s_d'], d['config']['k'], d['clocks']['sm_mhz'])
c=d['comparison']
for k in ('aggregated_chunked_at_slo','partitioned_optimizer','partitioned_boundary_aware'):
    v=c.get(k)
    if v: print(k, round(v['tok_s']), round(v['window_ms'],1), v['k'], round(v.get('tbt_max_ms',0),1), v.get('sm_mhz'))
print(json.dumps(d['roofline'])[:500])
print(d['kernel_timing'])
PY
