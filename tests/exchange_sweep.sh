# bench.py at NG GPUs: allgather exchange vs owner vote
run() { # label env...
  label=$1; shift
  env "$@" python -m torch.distributed.run --nnodes=1 --nproc-per-node=$NG --master-addr=127.0.0.1 --master-port=$((29500 + RANDOM % 1000)) bench.py --gpus $NG --steps 50 --warmup 5 --no-e2e --workload $WL 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$label', d['config']['workload'], d['n_gpus'], round(d['ms_per_step'],4), round(d['step_roofline']['frac'],3), {k:round(v['avg_ms'],4) for k,v in d['kernels'].items()})"
}
for WL in ${WLS:-gpt2s_sumsigns tinyllama_1bit}; do
run owner-vote LIONCUB_AG_MAX_P=1
run allgather LIONCUB_AG_MAX_P=64
done
