# round 2: CTA-pair split-K — op tests (short timeout first), layer suite, cfg3 bench + sweep
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "op_gemm" 2>&1 | tail -3
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/tests_splitk.log; cat gpurun_out/tests_splitk.log
timeout 1800 python bench.py --steps 10 --warmup 3 --sweep > gpurun_out/bench_cfg3_e.json 2> gpurun_out/bench_cfg3_e.log
grep -E "split:|timed:|sweep S_d=(48|56|64|72)" gpurun_out/bench_cfg3_e.log
python - <<'PY'
import json
d=json.load(open('gpurun_out/bench_cfg3_e.json'))
print(d['value'], d['ms_per_step'], d['config']['s_d'], d['config']['k'], d['clocks']['sm_mhz'])
c=d['comparison']
for k in ('aggregated_chunked_at_slo','partitioned_optimizer','partitioned_boundary_aware'):
    v=c.get(k)
    if v: print(k, round(v['tok_s']), round(v['window_ms'],1), v['k'], round(v['t_decode_ms']/v['k'],1), round(v.get('tbt_max_ms',0),1), v.get('sm_mhz'))
print(d['kernel_seconds_per_step'])
PY
