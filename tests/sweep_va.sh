# vote/update kernel variants at P = N on the TinyLlama layout (gpurun --gpus N)
set -u
N=${1:-4}
VARIANTS=${2:-"default share4 default share4"}
for v in $VARIANTS; do
  if [ $v = default ]; then unset LIONCUB_LIB; else export LIONCUB_LIB=$PWD/paper_2411_16462_b200/_lib/liblioncub_$v.so; fi
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 \
    --master-port=29615 bench.py --gpus $N --workload tinyllama_1bit --steps 50 --warmup 5 \
    --no-cpu-baseline --no-e2e > gpurun_out/va.json 2> /dev/null
  python -c "import json; d=json.loads(open('gpurun_out/va.json').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],3), {k: round(v['avg_ms'],3) for k,v in d['kernels'].items()})"
done
