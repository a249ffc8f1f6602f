mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:"gemm2" -c 4 -o gpurun_out/gemm2_full python bench.py --profile-only --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_g2.log 2>&1
ls -la gpurun_out/gemm2_full.ncu-rep
