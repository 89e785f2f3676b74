# A/B of the fused-sync variants on one multi-GPU box (gpurun --gpus N)
set -u
N=${1:-4}
for mode in serial side inline; do
  export LIONCUB_SYNC_MEAN=$mode
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 \
    --master-port=29611 bench.py --gpus $N --workload flat7b_1bit_sync --steps 10 --warmup 3 \
    --no-cpu-baseline --no-e2e > gpurun_out/sw_${mode}_n$N.json 2> gpurun_out/sw_${mode}_n$N.err
  python -c "import json; d=json.loads(open('gpurun_out/sw_${mode}_n$N.json').read().strip().splitlines()[-1]); print('$mode', round(d['ms_per_step'],2), {k: round(v['avg_ms'],2) for k,v in d['kernels'].items()})"
done
