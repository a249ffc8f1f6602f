# round 2: prefill attention softmax with prefetched TMEM loads and deferred store waits — parity, timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity_deep.py tests/test_gpu_parity.py -x -q -k "prefill or cfg2 or tiny or mini or corun or graph" 2>&1 | tail -3
for i in 1 2; do
timeout 600 python tools/prefill_attn_bench.py --variants DUET_FA_PERSIST=1 --sms 84,148 2>&1 | grep -v "^$"
done | tee gpurun_out/fa_ld_ab.txt
DUET_FA_TRACE=1 timeout 300 python tools/prefill_attn_bench.py --child --sms 148 2>&1 | grep FA_TRACE | head -20 > gpurun_out/fa_ld_trace.txt
