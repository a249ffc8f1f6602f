mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "${TESTK:-parity}" 2>&1 | tail -5
timeout 600 ncu --clock-control none --metrics gpu__time_duration.sum -k regex:"fa_tc|gemm_tc|decode_tc" --csv --profile-from-start off python bench.py --profile-only --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/fa_times.csv 2>/dev/null
python tools/ncu_times.py gpurun_out/fa_times.csv
DUET_FA_TRACE=1 timeout 300 python bench.py --profile-only --steps 1 --warmup 1 --no-cpu-baseline 2>/dev/null | grep FA_TRACE | head -12
