# Bench lines of every config on one box (developer script; outputs under
# gpurun_out/): config 3 (default), 1 (fp32, one-CTA step), 2 (bf16x2 fused),
# 4 (dense tf32), and the reference arm at config 3.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.draw,power.limit --format=csv > gpurun_out/gpu_info.txt
for c in 3 1 2 4; do
  timeout 600 python bench.py --config $c > gpurun_out/bench_cfg$c.json 2> gpurun_out/bench_cfg$c.err; echo "bench config $c exit $?"
  python -c "import json; d=json.loads(open('gpurun_out/bench_cfg$c.json').read().strip().splitlines()[-1]); print($c, d['value'], d['unit'], d['ms_per_step']*1e3, 'us/step', 'frac', d['roofline']['frac'], d['clocks']['sm_mhz'])"
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo "reference exit $?"
