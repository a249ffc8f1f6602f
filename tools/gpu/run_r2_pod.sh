# round 2 (late): fused POD attention (f4) — parity, then the cfg2 temporal step with / without it
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "cfg2_full or forced_attention or llama_shapes or qwen or running_max" 2>&1 | tail -3
for i in 1 2; do
for v in 1 0; do
  DUET_POD=$v timeout 900 python bench.py --config cfg2 --steps 50 --warmup 5 --no-cpu-baseline > /tmp/b.json 2>/dev/null
  python -c "
import json; d=json.load(open('/tmp/b.json'))
print('POD=$v', round(d['value']), 'ms/step %.4f' % d['ms_per_step'], 'corun', d['config'].get('attention_corun_s_d'), 'mhz', d['clocks']['sm_mhz'])"
done
done | tee gpurun_out/pod_ab.txt
