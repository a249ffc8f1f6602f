mkdir -p gpurun_out
timeout 600 python tools/ar_bench.py --out gpurun_out/f3_ar_bench.txt 2>&1 | tail -12
