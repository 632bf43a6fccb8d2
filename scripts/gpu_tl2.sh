timeout 300 python scripts/fused_timeline.py 3 bf16x2 2>&1 | grep -v "^ *\(10\|12\|2[78]\) " | tail -14
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "forced_m_tiles or fused or bf16x2" 2>&1 | tail -2
