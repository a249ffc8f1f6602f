# round 2 (late): ncu --set full of the persistent prefill attention at q = 8192 (full device), then the default cfg3 bench
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fa_tc_kernel" \
  --launch-skip 26 --launch-count 1 -o gpurun_out/ncu_fa_persist -f python tools/prefill_attn_bench.py --child --sms 148 \
  > gpurun_out/ncu_fa_persist.log 2>&1
tail -2 gpurun_out/ncu_fa_persist.log
timeout 1800 python bench.py > gpurun_out/bench_cfg3_i.json 2> gpurun_out/bench_cfg3_i.log
python - <<'PY'
import json
d=json.load(open('gpurun_out/bench_cfg3_i.json'))
print(d['value'], d['ms_per_step'], d['config']['s_d'], d['config']['k'], d['clocks']['sm_mhz'], d['roofline']['frac'])
c=d['comparison']
for k in ('aggregated','aggregated_chunked_at_slo','partitioned_optimizer','partitioned_boundary_aware'):
    v=c.get(k)
    if v: print(k, round(v['tok_s']), round(v['window_ms'],1), v['k'], round(v.get('tbt_median_ms',0),1), round(v.get('tbt_max_ms',0),1), v.get('sm_mhz'))
print(json.dumps(d['predictor']['per_side']))
print(d['kernel_seconds_per_step'])
PY
