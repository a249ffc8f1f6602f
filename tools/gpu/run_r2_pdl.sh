# round 2: split-unit target below 74; PDL on / off on the cfg3 spatial step at a fixed split (S_d = 56, k = 4)
mkdir -p gpurun_out
for u in 56 37; do
  DUET_GEMM2_SPLIT_UNITS=$u timeout 900 python tools/partition_bench.py --config cfg3-fit --only decode --sd 56 --reps 3 \
    --out gpurun_out/part_u${u}_56.json > /dev/null 2>&1
  python3 -c "
import json; d=json.load(open('gpurun_out/part_u${u}_56.json')); r=d['rows'][0] if 'rows' in d else d
print('units $u S_d 56', 't_step %.2f ms' % r['t_meas_ms'], 'gemm_decode %.1f us/launch' % (r['kernels']['gemm_decode']['s_per_launch']*1e6))"
done
for pdl in 1 0; do
  DUET_PDL=$pdl timeout 1200 python bench.py --steps 10 --warmup 3 --split 56,4 --no-cpu-baseline > gpurun_out/bench_pdl$pdl.json 2> gpurun_out/bench_pdl$pdl.log
  python3 -c "
import json; d=json.load(open('gpurun_out/bench_pdl$pdl.json')); v=d['comparison']['partitioned_optimizer']
print('PDL $pdl', 'value %.0f' % d['value'], 'window %.1f t_d/step %.2f t_p %.1f' % (v['window_ms'], v['t_decode_ms']/v['k'], v['t_prefill_ms']), 'mhz', v['sm_mhz'], 'dec_attn avg us', round(d['roofline']['avg_launch_us'],1), d['roofline']['kernel'])"
done
