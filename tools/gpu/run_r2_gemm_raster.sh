# grouped rasterization of the CTA-pair GEMM: op / layer parity, then the cfg3 bench (co-run calibration)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_deep.py -m gpu -x -q \
  -k "op_gemm or llama or qwen or stack or cfg2_full" 2>&1 | tail -5 > gpurun_out/raster_tests.log
cat gpurun_out/raster_tests.log
timeout 1200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg3_r.json 2> gpurun_out/bench_cfg3_r.log
tail -4 gpurun_out/bench_cfg3_r.log
