# round 2: FA K/V ring depths — parity with the new default, then timing of the variants
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity_deep.py tests/test_gpu_parity.py -m gpu -x -q -k "prefill_attention or cfg2_full" 2>&1 | tail -2
timeout 600 python tools/prefill_attn_bench.py --variants DUET_FA_RING=2x3,DUET_FA_RING=3x2 --sms 84,148 --out gpurun_out/fa_ring.json 2>&1 | tee gpurun_out/fa_ring.txt
