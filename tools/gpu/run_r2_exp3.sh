# round 2: legacy HMMA rate probe; ncu full capture of the decode attention (cfg3 batch, full device, cp4x2)
mkdir -p gpurun_out
./tools/probes/bin/probe_hmma | tee gpurun_out/probe_hmma.txt
DUET_DECODE=cp4x2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_tc -c 2 -o gpurun_out/ncu_decode_cfg3 -f python tools/decode_attn_bench.py --child --sms 148 > gpurun_out/ncu_decode.log 2>&1
tail -3 gpurun_out/ncu_decode.log
( time timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_smoke3.csv python -c "import __graft_entry__ as g; g.smoke()" ) > gpurun_out/smoke_ncu3.log 2>&1
echo "ncu smoke rc=$?"; grep -v "^==PROF==" gpurun_out/smoke_ncu3.log | tail -4
