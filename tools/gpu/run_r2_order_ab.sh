# round 2 (late): decode attention CTAs longest-context-first (DUET_DECODE_ORDER=1, default) vs request order
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity_deep.py tests/test_gpu_parity.py -x -q -k "decode or spatial or temporal or lm_head" 2>&1 | tail -3
for i in 1 2; do
for v in 0 1; do
  DUET_DECODE_ORDER=$v timeout 600 python tools/decode_attn_bench.py --variants cp4x2 --sms 48,56,64,148 2>&1 | grep cfg3 | sed "s/^/ORDER=$v /"
done
done | tee gpurun_out/order_ab.txt
for v in 0 1; do
  DUET_DECODE_ORDER=$v timeout 1200 python bench.py --split 56,4 --steps 20 --warmup 3 --no-cpu-baseline > /tmp/b.json 2>/dev/null
  python -c "
import json; d=json.load(open('/tmp/b.json')); c=d['comparison']['partitioned_optimizer']
print('ORDER=$v', round(d['value']), 'window %.1f t_d %.1f t_p %.1f mhz %s' % (c['window_ms'], c['t_decode_ms'], c['t_prefill_ms'], c['sm_mhz']))"
done | tee -a gpurun_out/order_ab.txt
