# functional check of the multi-rank bench path on one GPU (2 ranks, gloo); not a measurement
GEIG_BENCH_SHARE_GPU=1 GEIG_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --spinup 0 > gpurun_out/mr.json 2> gpurun_out/mr.err
echo "multi-rank exit $?"; tail -c 1500 gpurun_out/mr.json; tail -5 gpurun_out/mr.err
timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/b1.json 2>gpurun_out/b1.err; echo "bench1 exit $?"; python -c "
import json;d=json.loads(open('gpurun_out/b1.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['e2e'])"
