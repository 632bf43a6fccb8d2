mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.draw,power.limit --format=csv > gpurun_out/gpu_info.txt
python -c "from paper_2206_04993_b200 import build; build.build(force=True)" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?"; tail -1 gpurun_out/smoke.log
timeout 1200 bash scripts/gpu_abfiles.sh > gpurun_out/ab.log 2>&1; echo "ab exit $?"; cat gpurun_out/ab.log | grep -E "^(new|old)|median"
