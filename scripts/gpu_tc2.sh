mkdir -p gpurun_out
timeout 120 python scripts/tc_probe.py tf32 > gpurun_out/tc_probe_tf32.log 2>&1; echo "probe tf32 exit $?"
cat gpurun_out/tc_probe_tf32.log | tail
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_bf16.log 2>&1; echo "bench exit $?"
tail -c 2500 gpurun_out/bench_bf16.log
