mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/pytest_gpu4.log 2>&1; echo "pytest exit $?"
tail -15 gpurun_out/pytest_gpu4.log
timeout 300 python scripts/phase_probe.py 3 bf16 2>&1 | tail -5
timeout 300 python scripts/phase_probe.py 2 bf16 2>&1 | tail -5
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_bf16_4.log 2>&1; echo "bench exit $?"
tail -c 1800 gpurun_out/bench_bf16_4.log
