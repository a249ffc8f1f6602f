# round 2: FA softmax with paired TMEM loads — parity, then timing (one-CTA and pair)
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity_deep.py -m gpu -x -q -k "prefill_attention" 2>&1 | tail -2
DUET_FA2=1 timeout 300 python -m pytest tests/test_gpu_parity_deep.py -m gpu -x -q -k "prefill_attention" 2>&1 | tail -2
timeout 600 python tools/prefill_attn_bench.py --variants DUET_FA2=0,DUET_FA2=1 --sms 84,148 --out gpurun_out/fa_ld.json 2>&1 | tee gpurun_out/fa_ld.txt
