timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_gpu.log
python scripts/ab.py 3 "A=1" | tail -1
python bench.py --steps 300 --warmup 10 --no-cpu-baseline --no-e2e --adam | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('adam', round(d['ms_per_step']*1e3,2))"
