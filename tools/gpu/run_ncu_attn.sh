mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:fa_tc -c 1 -o gpurun_out/fa_tc python bench.py --profile-only --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_fa.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:decode_tc -c 1 -o gpurun_out/dec24b python tools/partition_bench.py --only decode --sd 24 --reps 1 > gpurun_out/ncu_dec.log 2>&1
ls -la gpurun_out/*.ncu-rep
