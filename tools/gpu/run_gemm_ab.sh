mkdir -p gpurun_out
for cfg in "1 1" "0 1" "1 0" "0 0"; do
  set -- $cfg
  DUET_SPLITK=$1 DUET_GEMM_PF=$2 timeout 300 ncu --clock-control none --metrics gpu__time_duration.sum -k regex:"gemm_tc|decode_tc" -c 5 --csv python tools/partition_bench.py --only decode --sd ${SD:-24} --reps 1 > gpurun_out/gemm_ab_$1$2.csv 2>/dev/null
done
python tools/ncu_times.py gpurun_out/gemm_ab_*.csv
