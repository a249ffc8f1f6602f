# quick GPU check: parity tests (selected by $1 pattern) + decode partition sweep
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q ${1:+-k "$1"} 2>&1 | tail -15 > gpurun_out/tests.log
cat gpurun_out/tests.log
timeout 600 python tools/partition_bench.py --only decode --out gpurun_out/part_decode.json > gpurun_out/part_decode.log 2>&1
python - <<'PY'
import json
d=json.load(open('gpurun_out/part_decode.json'))
for r in d['rows']:
    print(r['side'], r['sms'], 'meas', round(r['t_meas_ms'],3), 'roof', round(r['t_roofline_ms'],3), 'frac', round(r['frac_of_roofline'],3), 'B', round(r['B_GBs']), {k:(round(v['s_per_launch']*1e6,1), round(v['gbs'])) for k,v in r['kernels'].items()})
PY
timeout 600 python bench.py --steps 50 --warmup 5 --sweep > gpurun_out/bench.log 2>&1
tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value',d['value'],'ms',d['ms_per_step'],'clk',d['clocks']); print('cmp',json.dumps(d.get('comparison',{}))[:600]); print('roof',d['roofline']); print('ks',d['kernel_seconds_in_timed_region'])"
