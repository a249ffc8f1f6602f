# round 2: launch list of the cfg3 timed region (profiler start/stop in bench.py) + ncu --set full of one
# decode-attention launch and one prefill GEMM launch of that region
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/launches_cfg3.csv python bench.py --profile-only --steps 1 --warmup 1 --no-cpu-baseline \
  > gpurun_out/ncu_cfg3_launches.log 2>&1
echo "launch list rc=$?"; wc -l gpurun_out/launches_cfg3.csv
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"decode_tc|gemm2" -c 3 \
  -o gpurun_out/ncu_cfg3_full -f python bench.py --profile-only --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_cfg3_full.log 2>&1
echo "full rc=$?"; tail -3 gpurun_out/ncu_cfg3_full.log
