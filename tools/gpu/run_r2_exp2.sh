# round 2: decode attention load-path A/B (bulk copies of pre-swizzled pages, early stage refill); timing only
mkdir -p gpurun_out
timeout 1200 python tools/decode_attn_bench.py --variants ${VARIANTS:-cp4x2,cp4x2e,bk4x2,bk4x2e,bk4x3e,bk8x2e,bk2x2e,bk4x3x2} --sms 16,32,48,64,148 --out gpurun_out/dec_bk.json 2>&1 | tee gpurun_out/dec_bk.txt
( time timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_smoke2.csv python -c "import __graft_entry__ as g; g.smoke()" ) > gpurun_out/smoke_ncu2.log 2>&1
echo "ncu smoke rc=$?"; grep -v "^==PROF==" gpurun_out/smoke_ncu2.log | tail -8
