mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q --timeout 200 -k "fused" > gpurun_out/pytest_fused.log 2>&1; echo "pytest exit $?"
tail -3 gpurun_out/pytest_fused.log
timeout 300 python scripts/phase_probe.py 3 bf16 2>&1 | tail -5
