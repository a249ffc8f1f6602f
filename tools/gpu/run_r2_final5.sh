# round 2 (final): full GPU suite, smoke, cfg2 line
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -8 > gpurun_out/tests_final5.log; cat gpurun_out/tests_final5.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py --config cfg2 --steps 50 --warmup 5 > gpurun_out/bench_cfg2_k.json 2> gpurun_out/bench_cfg2_k.log
python3 -c "import json; d=json.load(open('gpurun_out/bench_cfg2_k.json')); print('cfg2', d['value'], d['ms_per_step'], d['roofline']['frac'], d['config'].get('attention_corun_s_d'))"
