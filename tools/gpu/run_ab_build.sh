# A/B of a compile-time switch on the same box: bench with the default build, then with $EXTRA
mkdir -p gpurun_out
b() { timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['ms_per_step'], round(d['value']), round(d['roofline']['frac'],3), round(d['comparison'].get('partitioned_optimizer',{}).get('tok_s',0)))"; }
b A1; b A1
DUET_NVCC_EXTRA="$EXTRA" python -c "from paper_2511_04791_b200 import build as B; B.build()" > /dev/null 2>&1
b B1; b B1
python -c "from paper_2511_04791_b200 import build as B; B.build()" > /dev/null 2>&1
b A2
