# sanity of the restored tree + L2 re-read microbenchmark
mkdir -p gpurun_out
timeout 120 ./scripts/l2_mix > gpurun_out/l2_mix.txt 2>&1; echo "l2_mix exit $?"
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err; echo "bench exit $?"
cat gpurun_out/l2_mix.txt
