mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:fa_tc -c 1 -o gpurun_out/fa_tc python bench.py --profile-only --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_fa.log 2>&1
