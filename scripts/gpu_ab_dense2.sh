# same-box interleaved A/B of the working tree (new) against gpurun_in/ (old)
# on the config-4 dense step timing (scripts/dense_time.py tf32 3xtf32)
rm -rf /tmp/csrc_new; cp -r paper_2206_04993_b200/csrc /tmp/csrc_new
for r in 1 2; do
  for v in new old; do
    if [ $v = new ]; then cp /tmp/csrc_new/* paper_2206_04993_b200/csrc/; else cp gpurun_in/* paper_2206_04993_b200/csrc/; fi
    python -c "from paper_2206_04993_b200 import build; build.build(force=True)"
    echo "== $v"; timeout 300 python scripts/dense_time.py tf32 | head -1
  done
done
cp /tmp/csrc_new/* paper_2206_04993_b200/csrc/
