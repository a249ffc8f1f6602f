mkdir -p gpurun_out
for m in ${MODES:-1}; do
echo "== DUET_FA_TRACE=$m"
DUET_FA_TRACE=$m timeout 300 python bench.py --profile-only --steps 1 --warmup 1 --no-cpu-baseline 2>/dev/null | grep FA_TRACE | head -14
done
