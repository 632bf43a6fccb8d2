mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_convergence.py -q -s --timeout 300 > gpurun_out/pytest_conv.log 2>&1; echo "pytest exit $?"
grep -E "variant|config 0|passed|failed|Error" gpurun_out/pytest_conv.log | tail -10
