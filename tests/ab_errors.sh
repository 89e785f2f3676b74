# A/B of the strict (step) vs deferred error mode on one box (gpurun --gpus N)
N=${1:-2}
for w in ${WL:-tinyllama_1bit tinyllama_1bit_sync}; do
for mode in step deferred step; do
  LIONCUB_ERRORS=$mode timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 \
    --master-port=29621 bench.py --gpus $N --workload $w --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2> gpurun_out/ab.err
  python -c "import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); print('$w', '$mode', round(d['ms_per_step'],3), {k: round(v['avg_ms'],3) for k,v in d['kernels'].items()}, d['clocks']['sm_mhz'])"
done; done
