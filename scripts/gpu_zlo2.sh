GEIG_NO_ZLO=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "bf16x2_fp32_level_parity" 2>&1 | grep -E "^E .*parity errors|assert step" | head -8
GEIG_NO_ZLO=1 timeout 900 python -m pytest tests/test_gpu_convergence.py -m gpu -q -s -k "bf16x2" 2>&1 | grep -E "angles|passed|failed"
