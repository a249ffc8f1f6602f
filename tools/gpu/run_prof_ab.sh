# cost of the live per-launch CUDA-event timing inside the timed region
b() { timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['ms_per_step'],4), round(d['value']), round(d['e2e']['value']), d['roofline'].get('frac'), d['clocks'], d['predictor']['t_meas_ms'])"; }
b prof; DUET_BENCH_NOPROF=1 b noprof; b prof; DUET_BENCH_NOPROF=1 b noprof
