# round 2: does ncu run the spatial cfg3 step (green contexts)?  launch list + test rerun
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_profile.py -m gpu -x -q 2>&1 | tail -15
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_cfg3.csv \
  python bench.py --profile-only --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_cfg3_launches.log 2>&1
echo "ncu rc=$?"
grep -v "^==PROF== Profiling" gpurun_out/ncu_cfg3_launches.log | tail -15
wc -l gpurun_out/launches_cfg3.csv
