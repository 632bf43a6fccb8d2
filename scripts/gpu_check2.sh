mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -k "bf16 or tf32 or config1 or ragged_fp32 or dense_config0_traj" > gpurun_out/pytest_gpu2.log 2>&1; echo "pytest exit $?"
tail -25 gpurun_out/pytest_gpu2.log
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_bf16_2.log 2>&1; echo "bench exit $?"
tail -c 1500 gpurun_out/bench_bf16_2.log
