# round 2: four GEMM producer warps for the narrow tile — op parity, decode-side A/B, ncu of decode GEMMs
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "op_gemm or llama or cfg2_full" 2>&1 | tail -2
for pr in 2 4; do
  DUET_GEMM2_PROD=$pr timeout 900 python tools/partition_bench.py --config cfg3-fit --only decode --sd 56 --reps 3 \
    --out gpurun_out/part_prod$pr.json > gpurun_out/part_prod$pr.log 2>&1
  python3 -c "
import json; d=json.load(open('gpurun_out/part_prod$pr.json')); r=d['rows'][0] if 'rows' in d else d
print('prod $pr', 't_step %.2f ms' % r['t_meas_ms'], 'gemm_decode %.1f us/launch' % (r['kernels']['gemm_decode']['s_per_launch']*1e6))"
done
timeout 1200 ncu --set full --clock-control none --profile-from-start off -k regex:"gemm2" -c 6 \
  -o gpurun_out/ncu_cfg3_dgemm4 -f python bench.py --profile-only --steps 1 --warmup 1 --no-cpu-baseline --split 56,1 > gpurun_out/ncu_dgemm4.log 2>&1
python tools/ncu_summary.py gpurun_out/ncu_cfg3_dgemm4.ncu-rep
