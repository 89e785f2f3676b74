# vote/update variants incl. the fused-sync 7e9 step (gpurun --gpus 4)
VARIANTS=${VARIANTS:-"default"} bash tests/va_sweep3.sh
for v in ${VARIANTS:-default}; do
  if [ $v = default ]; then unset LIONCUB_LIB; else export LIONCUB_LIB=$PWD/paper_2411_16462_b200/_lib/liblioncub_$v.so; fi
  for wn in ${RUNS:-flat7b_1bit_sync:4:10 flat7b_1bit_sync:2:10 tinyllama_1bit:4:30 gpt2s_sumsigns:4:30}; do
    w=${wn%%:*}; rest=${wn#*:}; n=${rest%%:*}; st=${rest##*:}
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr=127.0.0.1 \
      --master-port=29615 bench.py --gpus $n --workload $w --steps $st --warmup 3 \
      --no-cpu-baseline --no-e2e > gpurun_out/va.json 2> /dev/null
    python -c "import json; d=json.loads(open('gpurun_out/va.json').read().strip().splitlines()[-1]); print('$v $w n=$n', round(d['ms_per_step'],3), {k: round(v['avg_ms'],3) for k,v in d['kernels'].items()}, d['clocks']['sm_mhz'])"
  done
done
