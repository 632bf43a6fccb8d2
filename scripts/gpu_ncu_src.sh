mkdir -p gpurun_out
python scripts/one_step.py 3 bf16x2 4 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"cca_step_kernel" -s 3 -c 1 -o gpurun_out/prof_src python scripts/one_step.py 3 bf16x2 4 > gpurun_out/ncu_src.log 2>&1
echo "full exit $?"; tail -3 gpurun_out/ncu_src.log
