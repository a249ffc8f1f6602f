# round profile: launch list of the timed bench steps + one `ncu --set full` capture of every hot kernel
mkdir -p gpurun_out
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_cfg2.csv python bench.py --profile-only --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off \
  -k regex:"gemm2|gemm_tc|fa_tc|decode_tc|splitk|rmsnorm|rope" -c 12 -o gpurun_out/prof_full_cfg2 \
  python bench.py --profile-only --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out/prof_full_cfg2.ncu-rep gpurun_out/launches_cfg2.csv
