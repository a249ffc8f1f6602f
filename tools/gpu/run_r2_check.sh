# round-2 check: the whole GPU suite, smoke(), a short default (cfg3) bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -25 > gpurun_out/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.log
cat gpurun_out/tests.log gpurun_out/smoke.log; tail -5 gpurun_out/bench_cfg3.log
