# side-stream fused-sync mean: CTA splits (gpurun --gpus N)
set -u
N=${1:-4}
export LIONCUB_SYNC_MEAN=side
for c in 3,1 2,1 2,2 4,1 1,2; do
  export LIONCUB_SYNC_SIDE_CTAS=$c
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 \
    --master-port=29614 bench.py --gpus $N --workload flat7b_1bit_sync --steps 10 --warmup 3 \
    --no-cpu-baseline --no-e2e > gpurun_out/ss_$c.json 2> /dev/null
  python -c "import json; d=json.loads(open('gpurun_out/ss_$c.json').read().strip().splitlines()[-1]); print('side $c', round(d['ms_per_step'],2), {k: round(v['avg_ms'],2) for k,v in d['kernels'].items()})"
done
