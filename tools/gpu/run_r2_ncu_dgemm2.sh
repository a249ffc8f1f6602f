# round 2 (late): ncu of the decode-side GEMMs (256-row batch on 56 SMs) after wide tiles + split-K
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --profile-from-start off -k regex:"gemm2" -c 12 \
  -o gpurun_out/ncu_cfg3_dgemm2 -f python bench.py --profile-only --steps 1 --warmup 1 --no-cpu-baseline --split 56,1 > gpurun_out/ncu_dgemm2.log 2>&1
echo "ncu rc=$?"
tail -3 gpurun_out/ncu_dgemm2.log
