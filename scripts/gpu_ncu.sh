# launch list (cold-cache, serialised) + one full capture of the top kernels
mkdir -p gpurun_out
CMD="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/ncu_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_list.log 2>&1
echo "list exit $?"
$CMD > gpurun_out/ncu_plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tc_gemm|update_kernel|zshuffle" -s 12 -c 4 -o gpurun_out/prof_r1 $CMD > gpurun_out/ncu_full.log 2>&1
echo "full exit $?"
tail -5 gpurun_out/ncu_full.log
