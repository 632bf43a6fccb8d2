timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_gpu.log
python scripts/ab.py 3 "A=1" | tail -1
cp gpurun_in/old_fused_step.cuh paper_2206_04993_b200/csrc/fused_step.cuh
python -c "from paper_2206_04993_b200 import build; build.build(force=True)"
echo old; python scripts/ab.py 3 "A=1" | tail -1
