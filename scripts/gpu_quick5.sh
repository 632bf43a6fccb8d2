mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/pytest_quick.log 2>&1; echo "pytest exit $?"
tail -3 gpurun_out/pytest_quick.log
timeout 300 python scripts/phase_probe.py 3 bf16 2>&1 | tail -5
