# round 2 (late): decode-attention variant inside the cfg3 partitioned window (co-run, power-capped clocks)
mkdir -p gpurun_out
for i in 1 2; do
for v in cp4x2 cp4x3x2 cp3x3 cp2x3; do
  DUET_DECODE=$v timeout 1200 python bench.py --split 56,4 --steps 20 --warmup 3 --no-cpu-baseline > /tmp/b.json 2>/dev/null
  python -c "
import json; d=json.load(open('/tmp/b.json')); c=d['comparison']['partitioned_optimizer']
print('DECODE=$v', round(d['value']), 'window %.1f t_d/step %.2f t_p %.1f mhz %s' % (c['window_ms'], c['t_decode_ms']/c['k'], c['t_prefill_ms'], c['sm_mhz']))"
done
done | tee gpurun_out/dec_variant_corun.txt
