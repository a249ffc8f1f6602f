# round 2: split-K work-unit target A/B on the decode side (cfg3-fit, S_d = 48 / 56 / 64)
mkdir -p gpurun_out
for u in 148 112 74; do
  for sd in 48 56 64; do
    DUET_GEMM2_SPLIT_UNITS=$u timeout 900 python tools/partition_bench.py --config cfg3-fit --only decode --sd $sd --reps 3 \
      --out gpurun_out/part_u${u}_$sd.json > /dev/null 2>&1
    python3 -c "
import json; d=json.load(open('gpurun_out/part_u${u}_$sd.json')); r=d['rows'][0] if 'rows' in d else d
print('units $u S_d $sd', 't_step %.2f ms' % r['t_meas_ms'], 'gemm_decode %.1f us/launch' % (r['kernels']['gemm_decode']['s_per_launch']*1e6))"
  done
done
