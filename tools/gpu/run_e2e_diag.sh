# where the e2e time goes: the pipelined host-buffer loop with one or both copy directions dropped,
# and with more / fewer hardware work queues
b() { timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['ms_per_step'],4), round(d['value']), round(d['e2e']['value']))"; }
for v in ${SKIPS:-none h2d d2h h2d,d2h}; do DUET_E2E_SKIP=$v b skip=$v; done
for c in ${CONNS:-}; do CUDA_DEVICE_MAX_CONNECTIONS=$c b conns=$c; done
