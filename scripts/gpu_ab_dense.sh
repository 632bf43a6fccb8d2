# same-session A/B of the working tree's update.cuh (new) against gpurun_in/update.cuh (old)
# on the config-4 dense step (scripts/dense_time.py tf32), interleaved builds (developer script)
rm -rf /tmp/upd_new; mkdir -p /tmp/upd_new; cp paper_2206_04993_b200/csrc/update.cuh /tmp/upd_new/
for r in 1 2; do
  cp /tmp/upd_new/update.cuh paper_2206_04993_b200/csrc/; python -c "from paper_2206_04993_b200 import build; build.build(force=True)"
  echo new; python scripts/dense_time.py tf32 | tail -2
  cp gpurun_in/update.cuh paper_2206_04993_b200/csrc/; python -c "from paper_2206_04993_b200 import build; build.build(force=True)"
  echo old; python scripts/dense_time.py tf32 | tail -2
done
cp /tmp/upd_new/update.cuh paper_2206_04993_b200/csrc/
