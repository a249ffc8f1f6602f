# round 2: narrow pair tile — full GPU suite, then cfg3 bench + sweep
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/tests_narrow.log
cat gpurun_out/tests_narrow.log
timeout 1800 python bench.py --steps 10 --warmup 3 --sweep > gpurun_out/bench_cfg3_sweep3.json 2> gpurun_out/bench_cfg3_sweep3.log
grep -E "split:|timed:|sweep S_d" gpurun_out/bench_cfg3_sweep3.log
