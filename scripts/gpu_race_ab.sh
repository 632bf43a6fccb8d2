# developer: failure counts of the multi-step fused launch at b = 100k (race hunt), dev-knob build
GEIG_NVCC_EXTRA="-DGEIG_DEV_KNOBS=1" python -c "from paper_2206_04993_b200 import build; build.build(force=True)" || exit 1
for v in "A=1" "GEIG_F_BARRIER=1" "GEIG_BU_BARRIER=1" "GEIG_NO_EARLY_COEF=1"; do
  echo "== $v"; env $v python scripts/race_probe.py 1 100000 64 8 3000 100 8 0.0086 2>&1 | grep -E "repeat [0-9]+:" | grep -vc "None"
done
