mkdir -p gpurun_out
set -x
timeout 600 python tools/partition_bench.py --only decode --out gpurun_out/part_decode.json > gpurun_out/part_decode.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:decode_tc|gemm_tc" -c 6 -o gpurun_out/dec24 python tools/partition_bench.py --only decode --sd 24 --reps 1 > gpurun_out/ncu_dec24.log 2>&1
python - <<'PY' > gpurun_out/part_summary.txt
import json
d=json.load(open('gpurun_out/part_decode.json'))
for r in d['rows']:
    print(r['side'], r['sms'], 'meas', round(r['t_meas_ms'],3), 'roof', round(r['t_roofline_ms'],3), 'frac', round(r['frac_of_roofline'],3), 'B', round(r['B_GBs']), {k:(round(v['s_per_launch']*1e6,1), round(v['gbs'])) for k,v in r['kernels'].items()})
PY
cat gpurun_out/part_summary.txt
