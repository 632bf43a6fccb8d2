# same-session A/B of the working tree (new) against files shipped in gpurun_in/ (old), interleaved builds
rm -rf /tmp/csrc_new; cp -r paper_2206_04993_b200/csrc /tmp/csrc_new
for r in 1 2; do
  cp /tmp/csrc_new/* paper_2206_04993_b200/csrc/; python -c "from paper_2206_04993_b200 import build; build.build(force=True)"
  echo new; python scripts/ab.py 2 "A=1" | tail -1
  cp gpurun_in/* paper_2206_04993_b200/csrc/; python -c "from paper_2206_04993_b200 import build; build.build(force=True)"
  echo old; python scripts/ab.py 2 "A=1" | tail -1
done
