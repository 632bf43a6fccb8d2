mkdir -p gpurun_out
timeout 300 python scripts/phase_probe.py 3 bf16 2>&1 | tail -8
timeout 300 python scripts/phase_probe.py 2 bf16 2>&1 | tail -8
timeout 300 python scripts/phase_probe.py 1 f32 2>&1 | tail -8
