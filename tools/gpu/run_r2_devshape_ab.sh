# round 2 (late): A/B shape-agnostic prefill graph (DUET_PREFILL_DEVSHAPE=1, default) vs per-shape graphs, cfg3 at a fixed split
mkdir -p gpurun_out
for i in 1 2; do
for v in 1 0; do
  DUET_PREFILL_DEVSHAPE=$v timeout 1200 python bench.py --split 64,4 --steps 20 --warmup 3 --no-cpu-baseline > /tmp/b.json 2>/dev/null
  python -c "
import json; d=json.load(open('/tmp/b.json')); c=d['comparison']['partitioned_optimizer']
print('DEVSHAPE=$v', round(d['value']), 'window %.1f t_d %.1f t_p %.1f mhz %s' % (c['window_ms'], c['t_decode_ms'], c['t_prefill_ms'], c['sm_mhz']))"
done
done | tee gpurun_out/devshape_ab.txt
