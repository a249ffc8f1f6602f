mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/tests.log; cat gpurun_out/tests.log
timeout 600 python bench.py --steps 50 --warmup 5 --sweep > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
tail -1 gpurun_out/bench_cfg2.json | cut -c1-400
timeout 900 python bench.py --config cfg3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
tail -3 gpurun_out/bench_cfg3.err; tail -1 gpurun_out/bench_cfg3.json | cut -c1-600
