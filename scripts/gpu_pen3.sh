timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_gpu.log | head -12
timeout 300 python scripts/fused_timeline.py 3 bf16x2 2>&1 | grep -E "^ +(21|22|14) "
bash scripts/gpu_abfiles.sh
