# decode-access-pattern bandwidth probe (register rings vs 1-D bulk copies) + the GPU test suite
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt 2>&1
timeout 300 tools/probes/bin/probe_decode_bw > gpurun_out/probe_decode_bw.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/tests.log
cat gpurun_out/probe_decode_bw.txt gpurun_out/tests.log
