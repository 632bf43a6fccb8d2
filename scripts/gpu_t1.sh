timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_gpu.log
bash scripts/gpu_ab.sh "A=1" 2>&1 | grep -v "^env"
