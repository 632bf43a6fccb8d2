# same-box interleaved A/B of the working tree (new) against files in
# gpurun_in/ (old) on the bench of the configs given as arguments
# (developer; prints median us/step per build and config)
rm -rf /tmp/csrc_new; cp -r paper_2206_04993_b200/csrc /tmp/csrc_new
CFGS="${@:-3}"
for r in 1 2 3; do
  for v in new old; do
    if [ $v = new ]; then cp /tmp/csrc_new/* paper_2206_04993_b200/csrc/; else cp gpurun_in/* paper_2206_04993_b200/csrc/; fi
    python -c "from paper_2206_04993_b200 import build; build.build(force=True)"
    for c in $CFGS; do
      timeout 300 python bench.py --config $c --steps 2000 --warmup 20 --spinup 0.3 --no-cpu-baseline --no-e2e 2>/dev/null | \
        python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v cfg $c', round(d['ms_per_step']*1e3, 2), d['clocks']['sm_mhz'])"
    done
  done
done
