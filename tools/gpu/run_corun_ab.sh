b() { DUET_BENCH_NOPROF=1 timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['ms_per_step'],4))"; }
for i in 1 2 3 4; do for v in -1 88 80; do DUET_CORUN=$v b corun=$v; done; done
