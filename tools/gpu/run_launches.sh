# launch list of the timed bench steps (ncu metrics-only pass); CORUN=0 for the sequential attention layout
mkdir -p gpurun_out
for v in ${CORUNS:-default 0}; do
  if [ "$v" = default ]; then e=""; else e="DUET_CORUN=$v"; fi
  env $e timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_cfg2_corun_$v.csv python bench.py --profile-only --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch_$v.log 2>&1
  python tools/ncu_times.py gpurun_out/launches_cfg2_corun_$v.csv
done
