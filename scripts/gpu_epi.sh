mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_gpu.log
bash scripts/gpu_ab.sh "A=1" "GEIG_TM=1" > gpurun_out/ab.txt 2>&1; cat gpurun_out/ab.txt
timeout 300 python scripts/fused_timeline.py 3 bf16x2 2>&1 | grep -v "^ *\(10\|12\|2[1-2]\|2[78]\) " | tail -14
