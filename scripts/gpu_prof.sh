# Bench + ncu evidence of the default configuration (developer script;
# outputs under gpurun_out/): the bench line, the launch list of the bench
# command (gpu__time_duration per launch) and one --set full capture of a
# single-step fused launch (per-step DRAM traffic for the roofline).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.draw,power.limit --format=csv > gpurun_out/gpu_info.txt
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench exit $?"
CMD="python bench.py --steps 5 --warmup 3 --spinup 0 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_small.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench.csv $CMD > gpurun_out/ncu_list_bench.log 2>&1
echo "list exit $?"
CMD2="python scripts/one_step.py 3 bf16x2 4"
$CMD2 > gpurun_out/plain_small2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"cca_step_kernel" -s 3 -c 1 -o gpurun_out/prof_final -f $CMD2 > gpurun_out/ncu_full_final.log 2>&1
echo "full exit $?"
