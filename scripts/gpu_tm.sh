mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_gpu.log
bash scripts/gpu_ab.sh "GEIG_TM=1" "A=1" > gpurun_out/tm.txt 2>&1
cat gpurun_out/tm.txt
timeout 300 python scripts/fused_timeline.py 3 bf16x2 2>&1 | tail -3
