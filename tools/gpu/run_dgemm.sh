mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "gemm" 2>&1 | tail -2
timeout 300 ncu --clock-control none --metrics gpu__time_duration.sum -k regex:"gemm_tc|splitk" -c 8 --csv python tools/partition_bench.py --only decode --sd 24 --reps 1 > gpurun_out/dg_times.csv 2>/dev/null
python tools/ncu_times.py gpurun_out/dg_times.csv
timeout 300 python tools/partition_bench.py --only decode --out gpurun_out/part_decode.json > /dev/null 2>&1
python - <<'PY'
import json
d=json.load(open('gpurun_out/part_decode.json'))
for r in d['rows']:
    print(r['sms'], 'meas', round(r['t_meas_ms'],3), {k:(round(v['s_per_launch']*1e6,1)) for k,v in r['kernels'].items()})
PY
