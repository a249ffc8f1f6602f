mkdir -p gpurun_out
for i in 1 2; do
timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('prof on ', d['ms_per_step'])"
DUET_BENCH_NOPROF=1 timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('prof off', d['ms_per_step'])"
done
