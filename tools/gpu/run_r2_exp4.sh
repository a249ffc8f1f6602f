# round 2: register-direct decode attention — op parity at full size + the layer tests, then timing
mkdir -p gpurun_out
for v in ${PV:-rg4p8 rg4}; do
  DUET_DECODE=$v timeout 900 python -m pytest tests/test_gpu_parity_deep.py tests/test_gpu_parity.py -m gpu -x -q \
    -k "decode_attention or llama or stack or tiny" 2>&1 | tail -3 > gpurun_out/rg_tests_$v.log
  echo "== $v"; cat gpurun_out/rg_tests_$v.log
done
timeout 1200 python tools/decode_attn_bench.py --variants ${VARIANTS:-cp4x2,rg4,rg4p4,rg4p8,rg4p16,rg2p8,rg8p8} --sms 16,32,48,64,148 --out gpurun_out/dec_rg.json 2>&1 | tee gpurun_out/dec_rg.txt
