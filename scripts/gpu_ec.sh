timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_gpu.log
python scripts/ab.py 3 "A=1" "GEIG_NO_EARLY_COEF=1" | tail -2
timeout 300 python scripts/fused_timeline.py 3 bf16x2 2>&1 | tail -2 | head -1
