timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "fused or run_cca or bf16x2" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_gpu.log
python scripts/ab.py 3 "A=1" "GEIG_CG_SYNC=1"
