mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_convergence.py -x -q -s --timeout 300 -k "bf16x2 or converges" > gpurun_out/pytest_x2.log 2>&1; echo "pytest exit $?"
grep -E "variant|passed|failed|Error|error" gpurun_out/pytest_x2.log | tail -12
