# developer: failure counts (dev build): phase U's tile barrier in the barrier region (default) vs in the ring (old)
GEIG_NVCC_EXTRA="-DGEIG_DEV_KNOBS=1" python -c "from paper_2206_04993_b200 import build; build.build(force=True)" || exit 1
for v in "A=1" "GEIG_DBG_MODE=8192"; do
  echo "== $v"; env $v python scripts/race_probe.py 1 100000 64 8 3000 100 8 0.0086 2>&1 | grep -E "repeat [0-9]+:" | grep -vc "None"
done
