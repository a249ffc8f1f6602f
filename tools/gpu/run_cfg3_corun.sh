# cfg3: bench with the co-run (sustained) calibration + the split sweep; decode / prefill sides alone
mkdir -p gpurun_out
timeout 1500 python bench.py --steps 10 --warmup 3 --sweep --no-cpu-baseline > gpurun_out/bench_cfg3_corun.json 2> gpurun_out/bench_cfg3_corun.log
tail -25 gpurun_out/bench_cfg3_corun.log
timeout 900 python tools/partition_bench.py --config cfg3-fit --only decode --sd 48 --reps 5 --out gpurun_out/part_cfg3_dec48.json > gpurun_out/part_cfg3.log 2>&1
timeout 900 python tools/partition_bench.py --config cfg3-fit --only decode --sd 64 --reps 5 --out gpurun_out/part_cfg3_dec64.json >> gpurun_out/part_cfg3.log 2>&1
tail -4 gpurun_out/part_cfg3.log
