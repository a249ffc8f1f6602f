# round 2: cfg3 bench with the smoothed / settled co-run calibration + sweep (predictor vs measured per split)
mkdir -p gpurun_out
timeout 1800 python bench.py --steps 10 --warmup 3 --sweep > gpurun_out/bench_cfg3_sweep2.json 2> gpurun_out/bench_cfg3_sweep2.log
grep -E "split:|timed:|sweep S_d" gpurun_out/bench_cfg3_sweep2.log
