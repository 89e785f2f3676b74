# vote/update kernel variants: single-GPU microbench, then multi-GPU bench lines
# (gpurun --gpus 4 -- VARIANTS="default simple" bash tests/va_sweep_mg.sh)
VARIANTS=${VARIANTS:-"default simple"} bash tests/va_sweep3.sh
for v in ${VARIANTS:-default simple}; do
  if [ $v = default ]; then unset LIONCUB_LIB; else export LIONCUB_LIB=$PWD/paper_2411_16462_b200/_lib/liblioncub_$v.so; fi
  for wn in ${RUNS:-tinyllama_1bit:4 tinyllama_1bit:2 gpt2s_sumsigns:4}; do
    w=${wn%%:*}; n=${wn##*:}
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr=127.0.0.1 \
      --master-port=29615 bench.py --gpus $n --workload $w --steps 30 --warmup 5 \
      --no-cpu-baseline --no-e2e > gpurun_out/va.json 2> /dev/null
    python -c "import json; d=json.loads(open('gpurun_out/va.json').read().strip().splitlines()[-1]); print('$v $w n=$n', round(d['ms_per_step'],3), {k: round(v['avg_ms'],3) for k,v in d['kernels'].items()}, d['clocks']['sm_mhz'])"
  done
done
