mkdir -p gpurun_out
CMD="python scripts/phase_probe.py 3 bf16"
$CMD > gpurun_out/plain_upd2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"update_res_kernel|cca_step_kernel" -s 4 -c 2 -o gpurun_out/prof_upd2 $CMD > gpurun_out/ncu_upd2.log 2>&1
echo "ncu exit $?"; tail -2 gpurun_out/ncu_upd2.log
