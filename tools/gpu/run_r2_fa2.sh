# round 2: CTA-pair flash attention — op parity first (short timeout), then timing vs the one-CTA kernel
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity_deep.py -m gpu -x -q -k "prefill_attention" 2>&1 | tail -3 > gpurun_out/fa2_tests.log
cat gpurun_out/fa2_tests.log
if grep -q passed gpurun_out/fa2_tests.log && ! grep -q failed gpurun_out/fa2_tests.log; then
  timeout 600 python -m pytest tests -m gpu -x -q -k "parity and (cfg2 or llama or stack or prefill or tiny or qwen)" 2>&1 | tail -3
  timeout 600 python tools/prefill_attn_bench.py --variants DUET_FA2=0,DUET_FA2=1 --sms 84,148 --out gpurun_out/fa2_bench.json 2>&1 | tee gpurun_out/fa2_bench.txt
fi
