# A/B of an environment switch: VAR=name, VALS="a b" (each run twice, interleaved)
b() { timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernel_seconds_per_step']; print('$1', round(d['ms_per_step'],4), round(d['value']), round(d['e2e']['value']), {a: round(v*1e6,1) for a,v in k.items()})"; }
for r in 1 2; do for v in $VALS; do env $VAR=$v bash -c "$(declare -f b); b $VAR=$v"; done; done
