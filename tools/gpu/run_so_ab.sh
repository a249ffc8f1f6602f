# interleaved A/B of two prebuilt libraries (tools/ab/libduet_A.so, libduet_B.so) on one box
b() { DUET_BENCH_NOPROF=1 timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['ms_per_step'],4), round(d['comparison'].get('partitioned_optimizer',{}).get('tbt_ms',0),4))"; }
for i in 1 2 3 4; do
  cp tools/ab/libduet_A.so paper_2511_04791_b200/libduet.so; b A
  cp tools/ab/libduet_B.so paper_2511_04791_b200/libduet.so; b B
done
