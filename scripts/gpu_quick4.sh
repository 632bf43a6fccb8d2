mkdir -p gpurun_out
timeout 300 python scripts/phase_probe.py 3 bf16 2>&1 | tail -5
timeout 300 python scripts/phase_probe.py 2 bf16 2>&1 | tail -5
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_fused.json 2>&1; echo "bench exit $?"
tail -c 1800 gpurun_out/bench_fused.json
