# round 2: FA exp2-emulation A/B + decode L2-prefetch A/B + parity of the defaults; smoke under ncu
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "prefill or cfg2 or decode_attention" 2>&1 | tail -4 > gpurun_out/exp1_tests.log
cat gpurun_out/exp1_tests.log
timeout 900 python tools/prefill_attn_bench.py --variants DUET_FA_EMU=0,DUET_FA_EMU=2,DUET_FA_EMU=3,DUET_FA_EMU=4 --sms 84,148 --out gpurun_out/fa_emu.json 2>&1 | tee gpurun_out/fa_emu.txt
timeout 900 python tools/decode_attn_bench.py --variants ${VARIANTS:-cp4x2,cp4x2p4,cp4x2p8,cp4x2p16,cp4x3x2p8} --sms 16,32,64,148 --out gpurun_out/dec_pf.json 2>&1 | tee gpurun_out/dec_pf.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_smoke.csv python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_ncu.log 2>&1
tail -3 gpurun_out/smoke_ncu.log
python tools/ncu_times.py gpurun_out/launches_smoke.csv | grep -v elementwise | head -20
