timeout 120 python scripts/one_step.py 3 bf16x2 5; echo "one_step exit $?"
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "run_cca or fused_step_bf16" > gpurun_out/pt1.log 2>&1; echo "pytest1 exit $?"; tail -2 gpurun_out/pt1.log
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python scripts/ab.py 3 "A=1" "GEIG_BU_BARRIER=1" | tail -2
