mkdir -p gpurun_out
CMD="python scripts/phase_probe.py 3 bf16"
$CMD > gpurun_out/plain_upd.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"update_kernel|tc_gemm" -s 6 -c 3 -o gpurun_out/prof_upd $CMD > gpurun_out/ncu_upd.log 2>&1
echo "ncu exit $?"; tail -3 gpurun_out/ncu_upd.log
