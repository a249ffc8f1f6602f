# round 2 (late): cfg3 with 2-SM (TPC) partition granularity vs the default 8-SM granularity, same box
mkdir -p gpurun_out
for g in fine default; do
  if [ $g = fine ]; then F=--fine-split; else F=; fi
  timeout 1800 python bench.py $F > gpurun_out/bench_cfg3_$g.json 2> gpurun_out/bench_cfg3_$g.log
  python - <<PY
import json
d=json.load(open('gpurun_out/bench_cfg3_$g.json'))
print('$g', round(d['value']), d['ms_per_step'], d['config']['s_d'], d['config']['k'], d['clocks']['sm_mhz'], d['config']['calibration_s'])
c=d['comparison']
for k in ('aggregated_chunked_at_slo','partitioned_optimizer','partitioned_boundary_aware'):
    v=c.get(k)
    if v: print(' ', k, round(v['tok_s']), round(v['window_ms'],1), v['k'], v.get('s_d'), round(v.get('t_decode_ms',0),1), round(v.get('t_prefill_ms',0),1), round(v.get('tbt_median_ms',0),1), round(v.get('tbt_max_ms',0),1), v.get('sm_mhz'))
print(' ', json.dumps(d['predictor']['per_side']))
PY
done
