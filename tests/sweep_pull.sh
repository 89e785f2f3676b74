# selective-sync fusion A/B on the TinyLlama layout (gpurun --gpus N)
set -u
N=${1:-4}
run() {
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 \
    --master-port=29618 bench.py --gpus $N --workload tinyllama_1bit_sync --steps 50 --warmup 5 \
    --no-cpu-baseline --no-e2e > gpurun_out/tl.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/tl.json').read().strip().splitlines()[-1]); print('$1', round(d['ms_per_step'],3))"
}
LIONCUB_SYNC_FUSE=all run separate
for c in 0 2 3 4; do LIONCUB_SYNC_PULL_VOTE_CAP=$c run pull_cap$c; done
LIONCUB_SYNC_FUSE=all run separate
