# round 2: split-K A/B on the decode side alone (cfg3 batch) at S_d = 56 / 64, same box; FA trace
mkdir -p gpurun_out
for sk in 0 1; do
  for sd in 56 64; do
    DUET_GEMM2_SPLITK=$sk timeout 900 python tools/partition_bench.py --config cfg3 --only decode --sd $sd --reps 3 \
      --out gpurun_out/part_sk${sk}_sd$sd.json > /dev/null 2>&1
    python - "$sk" "$sd" <<'PY'
import json,sys
d=json.load(open(f'gpurun_out/part_sk{sys.argv[1]}_sd{sys.argv[2]}.json'))
r=d['rows'][0] if 'rows' in d else d
k=r['kernels']
print('splitk', sys.argv[1], 'S_d', sys.argv[2], 't_step_ms %.2f' % r['t_meas_ms'], {n: round(v['s_per_launch']*1e6,1) for n,v in k.items()})
PY
  done
done
DUET_FA_TRACE=1 timeout 300 python tools/prefill_attn_bench.py --child --sms 148 2>/dev/null | grep FA_TRACE > gpurun_out/fa_trace.txt
grep -n "n_kt=64" gpurun_out/fa_trace.txt | head -2
