# round 2 (final): the default cfg3 bench twice back to back (spread on one box)
mkdir -p gpurun_out
for i in 1 2; do
  timeout 1800 python bench.py > gpurun_out/bench_cfg3_rep$i.json 2> gpurun_out/bench_cfg3_rep$i.log
  python - <<PY
import json
d=json.load(open('gpurun_out/bench_cfg3_rep$i.json'))
c=d['comparison']
print('rep$i', round(d['value']), 'S_d', d['config']['s_d'], 'k', d['config']['k'], 'mhz', d['clocks']['sm_mhz'],
      'chunked', round(c['aggregated_chunked_at_slo']['tok_s']), 'ratio %.3f' % (c['partitioned_optimizer']['tok_s'] / c['aggregated_chunked_at_slo']['tok_s']),
      'pred_err %.3f' % d['predictor']['per_side']['window'])
PY
done
