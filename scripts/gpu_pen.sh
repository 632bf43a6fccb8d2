for r in 1 2 3; do
  GEIG_NVCC_EXTRA="-DGEIG_PEN_REPS=$r" python -c "from paper_2206_04993_b200 import build; build.build(force=True)" || exit 1
  echo "reps $r"; timeout 300 python scripts/fused_timeline.py 3 bf16x2 2>&1 | grep -E "^ +(13|21|22|14) "
done
