mkdir -p gpurun_out
for m in ${MODES:-"" noload}; do
if [ "$m" = "none" ]; then unset DUET_FA_TRACE; else export DUET_FA_TRACE=$m; fi; timeout 300 ncu --clock-control none --metrics gpu__time_duration.sum -k regex:"fa_tc" --csv --profile-from-start off python bench.py --profile-only --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/fa_exp.csv 2>/dev/null
echo "mode=$m"; python tools/ncu_times.py gpurun_out/fa_exp.csv
done
if [ -n "$TESTK" ]; then timeout 900 python -m pytest tests -m gpu -x -q -k "$TESTK" 2>&1 | tail -2; fi
