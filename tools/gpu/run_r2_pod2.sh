# round 2 (final): fused POD launch role order A/B on the cfg2 temporal step (vs the green-context pair)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "pod" 2>&1 | tail -2
DUET_POD=1 DUET_POD_DEC_FIRST=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "cfg2_full" 2>&1 | tail -2
for i in 1 2; do
for v in "0 0" "1 0" "1 1"; do
  set -- $v
  DUET_POD=$1 DUET_POD_DEC_FIRST=$2 timeout 900 python bench.py --config cfg2 --steps 50 --warmup 5 --no-cpu-baseline > /tmp/b.json 2>/dev/null
  python -c "
import json; d=json.load(open('/tmp/b.json'))
print('POD=$1 DEC_FIRST=$2', round(d['value']), 'ms/step %.4f' % d['ms_per_step'], 'mhz', d['clocks']['sm_mhz'])"
done
done | tee gpurun_out/pod2_ab.txt
