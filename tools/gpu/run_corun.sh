# f4 co-run sweep: temporal cfg2 step with the two attentions side by side on an S_d / remainder split
mkdir -p gpurun_out
b() { timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernel_seconds_per_step']; print('corun=$1', round(d['ms_per_step'],4), round(d['value']), {a: round(v*1e6,1) for a,v in k.items()})"; }
for v in ${SWEEP:-0 32 48 64 80 96 0}; do DUET_CORUN=$v b $v; done
if [ -n "$TESTK" ]; then DUET_CORUN=${TESTV:-64} timeout 900 python -m pytest tests -m gpu -x -q -k "$TESTK" 2>&1 | tail -3; fi
