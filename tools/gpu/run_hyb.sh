# decode attention variants: parity (op-level at full size + layer tests) with the hybrid kernel forced,
# then the per-partition bandwidth table of every variant
mkdir -p gpurun_out
DUET_DECODE=hy4x3 timeout 900 python -m pytest tests/test_gpu_parity_deep.py tests/test_gpu_parity.py -m gpu -x -q \
  -k "decode_attention or llama or qwen or stack or tiny" 2>&1 | tail -8 > gpurun_out/hyb_tests.log
cat gpurun_out/hyb_tests.log
timeout 1200 python tools/decode_attn_bench.py --variants ${VARIANTS:-cp4x2,cp4x3x2,hy4x3,hy4x4,hy4x2,hy4x3x2,hy4x2x4,hy2x4} \
  --out gpurun_out/decode_attn_bench.json 2>&1 | tee gpurun_out/decode_attn_bench.txt
