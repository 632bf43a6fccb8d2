timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "tables" 2>&1 | tail -2
bash scripts/gpu_mr.sh 2>&1 | head -1
for r in 1 2; do
for f in "" "--split-step" "--split-step --no-tables"; do
  python bench.py --steps 1000 --warmup 20 --no-cpu-baseline --no-e2e $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f', round(d['ms_per_step']*1e3,2), 'us', d['config']['step'], d['roofline']['phases'] if 'products_ms' in d['roofline']['phases'] else '')"
done; done
