mkdir -p gpurun_out
timeout 120 python scripts/tc_probe.py cca > gpurun_out/tc_probe_cca.log 2>&1; echo "probe cca exit $?"
timeout 120 python scripts/tc_probe.py dense > gpurun_out/tc_probe_dense.log 2>&1; echo "probe dense exit $?"
cat gpurun_out/tc_probe_cca.log gpurun_out/tc_probe_dense.log | tail -30
