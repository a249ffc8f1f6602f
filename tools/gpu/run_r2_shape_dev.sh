# round 2 (final): prefill attention enumerating the step's own shape in shape-agnostic graphs
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity_deep.py tests/test_gpu_parity.py -x -q -k "graph or prefill or spatial or mini or trace" 2>&1 | tail -3
timeout 1200 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > /tmp/b.json 2>/dev/null
python -c "
import json; d=json.load(open('/tmp/b.json')); c=d['comparison']
print(round(d['value']), d['config']['s_d'], d['config']['k'], d['clocks']['sm_mhz'], 'chunked', round(c['aggregated_chunked_at_slo']['tok_s']), 't_p', round(c['partitioned_optimizer']['t_prefill_ms'],1))"
