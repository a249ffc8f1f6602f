# round 2: 2-SM partition granularity bench; ncu of the decode-side GEMMs at S_d = 56 in the cfg3 step
mkdir -p gpurun_out
timeout 1800 python bench.py --steps 20 --warmup 3 --fine-split > gpurun_out/bench_cfg3_fine.json 2> gpurun_out/bench_cfg3_fine.log
grep -E "split:|timed:|calibrated" gpurun_out/bench_cfg3_fine.log
python - <<'PY'
import json
d=json.load(open('gpurun_out/bench_cfg3_fine.json'))
print(d['value'], d['ms_per_step'], d['config']['s_d'], d['config']['k'], d['clocks']['sm_mhz'])
c=d['comparison']
for k in ('aggregated_chunked_at_slo','partitioned_optimizer','partitioned_boundary_aware'):
    v=c.get(k)
    if v: print(k, round(v['tok_s']), round(v['window_ms'],1), v['k'], round(v['t_decode_ms']/v['k'],1), round(v.get('tbt_max_ms',0),1), v.get('sm_mhz'))
print(json.dumps(d['predictor']['per_side']))
PY
timeout 1200 ncu --set full --clock-control none --profile-from-start off -k regex:"gemm2|gemm2_reduce" -c 10 \
  -o gpurun_out/ncu_cfg3_dgemm -f python bench.py --profile-only --steps 1 --warmup 1 --no-cpu-baseline --split 56,1 > gpurun_out/ncu_dgemm.log 2>&1
echo "ncu rc=$?"
