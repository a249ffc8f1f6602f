# round 2 measurement (2): new GPU tests, cfg3 bench + sweep, full trace, decode side alone at S_d = 48/64
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity_deep.py -m gpu -x -q -k "prefill_graph or stack" 2>&1 | tail -3 > gpurun_out/tests_pg.log
cat gpurun_out/tests_pg.log
timeout 1800 python bench.py --steps 10 --warmup 3 --sweep > gpurun_out/bench_cfg3_sweep.json 2> gpurun_out/bench_cfg3_sweep.log
tail -4 gpurun_out/bench_cfg3_sweep.log
timeout 900 python tools/partition_bench.py --config cfg3-fit --only decode --sd 64 --reps 3 --out gpurun_out/part_cfg3_dec64.json > gpurun_out/part_cfg3.log 2>&1
tail -3 gpurun_out/part_cfg3.log
timeout 2400 python tools/trace_bench.py --n-req 48 --qps 40 --max-iters 8000 --out gpurun_out/trace_cfg4.json > gpurun_out/trace_cfg4.log 2>&1
tail -4 gpurun_out/trace_cfg4.log | cut -c1-300
