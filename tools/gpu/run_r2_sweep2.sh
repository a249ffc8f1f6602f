# round 2 (late): cfg3 split sweep with the final kernels (Fig. 7 / Fig. 8 table)
mkdir -p gpurun_out
timeout 2400 python bench.py --sweep --steps 20 --warmup 3 > gpurun_out/bench_cfg3_sweep_f.json 2> gpurun_out/bench_cfg3_sweep_f.log
python tools/render_sweep.py gpurun_out/bench_cfg3_sweep_f.json | head -30
