for v in 1 0 1 0; do
  GEIG_NVCC_EXTRA="-DGEIG_VARIANTS=$v" python -c "from paper_2206_04993_b200 import build; build.build(force=True)" || exit 1
  echo "variants $v"; python scripts/ab.py 2 "A=1" | tail -1
  timeout 300 python scripts/fused_timeline.py 3 bf16x2 2>&1 | tail -2 | head -1
done
