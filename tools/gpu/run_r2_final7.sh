# round 2 (final): full GPU suite + smoke on the final code
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -8 > gpurun_out/tests_final7.log; cat gpurun_out/tests_final7.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
