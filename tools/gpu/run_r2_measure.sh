# round 2 measurement: cfg3 bench with the split sweep (Fig. 7/8-style table), cfg2 bench line,
# trace-driven serving (static / static_slo / adaptive), and the env a profiled process sees
mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum -c 1 python -c "import os; print('ENV', sorted(k for k in os.environ if 'NV' in k or 'CUDA' in k or 'PRELOAD' in k or 'INJECT' in k))" 2>&1 | grep ENV > gpurun_out/ncu_env.txt
cat gpurun_out/ncu_env.txt
timeout 1800 python bench.py --steps 10 --warmup 3 --sweep > gpurun_out/bench_cfg3_sweep.json 2> gpurun_out/bench_cfg3_sweep.log
tail -30 gpurun_out/bench_cfg3_sweep.log
timeout 900 python bench.py --config cfg2 --steps 20 --warmup 5 > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.log
tail -3 gpurun_out/bench_cfg2.log
timeout 1500 python tools/trace_bench.py --n-req 48 --qps 40 --out gpurun_out/trace_cfg4.json > gpurun_out/trace_cfg4.log 2>&1
tail -5 gpurun_out/trace_cfg4.log | cut -c1-400
