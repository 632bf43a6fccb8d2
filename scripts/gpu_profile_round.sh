# Round profiling: bench line, ncu launch list of the same command, one full
# capture of the products kernels + update kernel (developer script).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu_info.txt
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench exit $?"
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_small.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench.csv $CMD > gpurun_out/ncu_list_bench.log 2>&1
echo "list exit $?"
$CMD > gpurun_out/plain_small2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tc_gemm|zshuffle|update_kernel" -s 8 -c 4 -o gpurun_out/prof_round $CMD > gpurun_out/ncu_full_round.log 2>&1
echo "full exit $?"
tail -c 600 gpurun_out/bench_default.json
