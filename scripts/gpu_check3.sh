mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/pytest_gpu3.log 2>&1; echo "pytest exit $?"
tail -25 gpurun_out/pytest_gpu3.log
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_bf16_3.log 2>&1; echo "bench exit $?"
tail -c 1500 gpurun_out/bench_bf16_3.log
