mkdir -p gpurun_out
bash scripts/gpu_ab.sh "A=1" "GEIG_DBG_MODE=2" "GEIG_DBG_MODE=1" "GEIG_DBG_MODE=3" "GEIG_DBG_NOSTORE=1" > gpurun_out/exp1.txt 2>&1
python bench.py --steps 1000 --warmup 20 --no-cpu-baseline --no-e2e --math bf16 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bf16', round(d['value']/1e6,2), 'M samples/s', round(d['ms_per_step']*1e3,1), 'us', {k:v for k,v in d['roofline']['phases'].items() if k!='source'})" >> gpurun_out/exp1.txt 2>&1
timeout 300 python scripts/fused_timeline.py 3 bf16x2 >> gpurun_out/exp1.txt 2>&1
GEIG_DBG_MODE=2 timeout 300 python scripts/fused_timeline.py 3 bf16x2 >> gpurun_out/exp1.txt 2>&1
cat gpurun_out/exp1.txt
