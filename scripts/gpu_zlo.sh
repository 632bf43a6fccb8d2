GEIG_NO_ZLO=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_convergence.py -m gpu -q -s -k "bf16x2 or fused or forced or random" 2>&1 | grep -E "passed|failed|FAILED|bf16x2 tcgen05|Alg. 3" | head -12
python scripts/ab.py 3 "A=1" "GEIG_NO_ZLO=1" | tail -2
