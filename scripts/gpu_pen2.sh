timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py -m gpu -q -x 2>&1 | tail -2
timeout 300 python scripts/fused_timeline.py 3 bf16x2 2>&1 | grep -E "^ +(21|22|14) "
bash scripts/gpu_abfiles.sh
