# round 2: decode-side GEMM tile width A/B at S_d = 56 (narrow default vs wide + split-K), producers 2
mkdir -p gpurun_out
for v in "0 2" "256 2" "128 2"; do
  set -- $v
  DUET_GEMM2_BN=$1 DUET_GEMM2_PROD=$2 timeout 900 python tools/partition_bench.py --config cfg3-fit --only decode --sd 56 --reps 3 \
    --out gpurun_out/part_bn$1.json > gpurun_out/part_bn$1.log 2>&1
  python3 -c "
import json; d=json.load(open('gpurun_out/part_bn$1.json')); r=d['rows'][0] if 'rows' in d else d
print('BN $1 prod $2', 't_step %.2f ms' % r['t_meas_ms'], 'gemm_decode %.1f us/launch' % (r['kernels']['gemm_decode']['s_per_launch']*1e6))"
done
