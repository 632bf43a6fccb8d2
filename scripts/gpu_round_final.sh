# Round deliverables on one GPU box: tests, smoke, bench lines (both arms),
# ncu launch list of the bench command and one full capture of the fused
# step kernel (developer script; outputs under gpurun_out/).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.draw,power.limit --format=csv > gpurun_out/gpu_info.txt
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?"; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench exit $?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo "reference exit $?"
CMD="python bench.py --steps 5 --warmup 3 --spinup 0 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_small.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench.csv $CMD > gpurun_out/ncu_list_bench.log 2>&1
echo "list exit $?"
# full capture of ONE single-step launch (per-step DRAM traffic for the roofline)
CMD2="python scripts/one_step.py 3 bf16x2 4"
$CMD2 > gpurun_out/plain_small2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"cca_step_kernel" -s 3 -c 1 -o gpurun_out/prof_final $CMD2 > gpurun_out/ncu_full_final.log 2>&1
echo "full exit $?"
tail -c 400 gpurun_out/bench_default.json
