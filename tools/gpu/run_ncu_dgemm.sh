mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"gemm_tc|splitk" -c 8 -o gpurun_out/dgemm24 python tools/partition_bench.py --only decode --sd 24 --reps 1 > gpurun_out/ncu_dgemm.log 2>&1
ls -la gpurun_out/dgemm24.ncu-rep
