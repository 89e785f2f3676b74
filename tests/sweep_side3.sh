# side-stream mean vs capped vote grid (va,mean CTAs/SM) for the 7e9 fused
# sync step after the vote/update redesign (gpurun --gpus 4)
N=${N:-4}
for c in ${CFGS:-2,1 2,2 3,1 1,1}; do
  LIONCUB_SYNC_SIDE_CTAS=$c timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N \
    --master-addr=127.0.0.1 --master-port=29631 bench.py --gpus $N --steps 10 --warmup 3 \
    --no-cpu-baseline --no-e2e > gpurun_out/side3.json 2> /dev/null
  python -c "import json; d=json.loads(open('gpurun_out/side3.json').read().strip().splitlines()[-1]); print('$c n=$N', round(d['ms_per_step'],3), {k: round(v['avg_ms'],3) for k,v in d['kernels'].items()})"
done
