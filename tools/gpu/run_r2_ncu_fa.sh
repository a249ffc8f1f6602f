# round 2: ncu --set full of the one-CTA and the CTA-pair flash attention at q = 8192 (full device)
mkdir -p gpurun_out
for v in 0 1; do
  DUET_FA2=$v timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fa2_kernel|fa_tc_kernel" \
    --launch-skip 26 --launch-count 1 -o gpurun_out/ncu_fa_v$v -f python tools/prefill_attn_bench.py --child --sms 148 \
    > gpurun_out/ncu_fa_v$v.log 2>&1
  tail -2 gpurun_out/ncu_fa_v$v.log
done
