# round 2: one-pass FA softmax + two-producer CTA-pair GEMM — parity, then A/Bs
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity_deep.py -m gpu -x -q -k "prefill_attention" 2>&1 | tail -2
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "op_gemm or cfg2_full or llama" 2>&1 | tail -2
timeout 600 python tools/prefill_attn_bench.py --variants DUET_FA_RING=3x2 --sms 84,148 2>&1 | tee gpurun_out/fa_onepass.txt
DUET_FA_TRACE=1 timeout 300 python tools/prefill_attn_bench.py --child --sms 148 2>/dev/null | grep FA_TRACE > gpurun_out/fa_trace2.txt
awk '/n_kt=64/{f=1} f' gpurun_out/fa_trace2.txt | sed -n 10,14p
for v in "1 1" "2 1" "2 0"; do
  set -- $v
  DUET_GEMM2_PROD=$1 DUET_GEMM2_SPLITK=$2 timeout 900 python tools/partition_bench.py --config cfg3-fit --only decode --sd 56 --reps 3 \
    --out gpurun_out/part_p$1_s$2.json > gpurun_out/part_p$1_s$2.log 2>&1
  tail -2 gpurun_out/part_p$1_s$2.log | cut -c1-400
done
