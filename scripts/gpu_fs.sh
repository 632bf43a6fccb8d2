timeout 120 python scripts/one_step.py 3 bf16x2 5; echo "one_step exit $?"
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_gpu.log | head -8
python scripts/ab.py 3 "A=1" "GEIG_NO_EARLY_B=1" | tail -2
timeout 300 python scripts/fused_timeline.py 3 bf16x2 2>&1 | grep -E "^ +(3|4|5|6|11|17|7) "
