# fused-sync mean placement at P = N (gpurun --gpus N)
set -u
N=${1:-2}
run() {
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 \
    --master-port=29614 bench.py --gpus $N --workload flat7b_1bit_sync --steps 8 --warmup 3 \
    --no-cpu-baseline --no-e2e > gpurun_out/s2.json 2> /dev/null
  python -c "import json; d=json.loads(open('gpurun_out/s2.json').read().strip().splitlines()[-1]); print('$1', round(d['ms_per_step'],2), {k: round(v['avg_ms'],2) for k,v in d['kernels'].items()})"
}
LIONCUB_SYNC_MEAN=serial run serial
for c in 1,3 1,2 2,2 2,4 1,6; do LIONCUB_SYNC_MEAN=side LIONCUB_SYNC_SIDE_CTAS=$c run side$c; done
