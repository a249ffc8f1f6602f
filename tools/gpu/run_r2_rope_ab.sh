# round 2: decode side (256-row batch) with the QKV GEMM's fused RoPE epilogue vs split-K QKV + separate RoPE pass
mkdir -p gpurun_out
for i in 1 2; do
for v in 1 0; do
  for sd in 56 64; do
    DUET_FUSE_ROPE=$v timeout 600 python tools/partition_bench.py --config cfg3-fit --only decode --sd $sd --reps 5 --out /tmp/pb.json > /dev/null 2>&1
    python -c "
import json; d=json.load(open('/tmp/pb.json')); r=d['rows'][0]; k=r['kernels']
print('FUSE_ROPE=$v', 'S_d', r['sms'], 't_step %.3f ms' % r['t_meas_ms'], ' '.join('%s %.1f us' % (n, v['s_per_launch']*1e6) for n, v in k.items()))"
  done
done
done | tee gpurun_out/rope_ab.txt
