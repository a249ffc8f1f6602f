mkdir -p gpurun_out
timeout 240 python -m pytest tests/test_gpu_parity.py -x -q -k "gemm" 2>&1 | tail -5
timeout 600 python -m pytest tests -m gpu -x -q -k "llama or cfg2 or tiny" 2>&1 | tail -3
timeout 300 ncu --clock-control none --metrics gpu__time_duration.sum -k regex:"gemm" --csv --profile-from-start off python bench.py --profile-only --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/g2_times.csv 2>/dev/null
python tools/ncu_times.py gpurun_out/g2_times.csv
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['ms_per_step'], d['roofline']['frac'], d['kernel_seconds_per_step'], d['comparison'].get('partitioned_optimizer'))"
