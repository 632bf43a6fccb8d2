for u in 4 1 2 8; do
  GEIG_NVCC_EXTRA="-DGEIG_PEN_UNROLL=$u" python -c "from paper_2206_04993_b200 import build; build.build(force=True)" || exit 1
  echo "unroll $u"; python scripts/ab.py 3 "A=1" | tail -1
done
