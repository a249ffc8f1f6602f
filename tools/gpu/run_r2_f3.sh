# round 2: fused GEMM + allreduce (f3) parity — emulated ranks, graph replay, single-rank ctx stacks
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_f3.py -x -q 2>&1 | tail -30 > gpurun_out/f3_tests.log
cat gpurun_out/f3_tests.log
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "op_gemm or tp_allreduce" 2>&1 | tail -3
