# developer: failure counts (dev build) with param-space maps for repeated batches vs forced global-memory maps
GEIG_NVCC_EXTRA="-DGEIG_DEV_KNOBS=1" python -c "from paper_2206_04993_b200 import build; build.build(force=True)" || exit 1
for v in "A=1" "GEIG_XMAPS_ALWAYS=1"; do
  echo "== $v"; env $v python scripts/race_probe.py 1 100000 64 8 3000 100 8 0.0086 2>&1 | grep -E "repeat [0-9]+:" | grep -vc "None"
done
