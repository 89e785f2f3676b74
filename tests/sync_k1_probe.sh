# K1 time with and without the (selective) momentum sync, and the pull vs
# separate sync (gpurun --gpus N -- bash tests/sync_k1_probe.sh N)
N=${1:-4}
for cfg in "tinyllama_1bit X=1" "tinyllama_1bit_sync X=1" "tinyllama_1bit_sync LIONCUB_SYNC_FUSE=0" "tinyllama_1bit_sync LIONCUB_ERRORS=deferred"; do
  set -- $cfg
  env $2 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 \
    --master-port=29617 bench.py --gpus $N --workload $1 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/k1.json 2> gpurun_out/k1.err
  python -c "import json; d=json.loads(open('gpurun_out/k1.json').read().strip().splitlines()[-1]); print('$1 $2', round(d['ms_per_step'],3), {k: (round(v['avg_ms'],3), v['launches']) for k,v in d['kernels'].items()}, d['clocks']['sm_mhz'])"
done
