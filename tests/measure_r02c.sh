# Round-2 final multi-GPU rows after the vote/update kernel redesign
# (gpurun --gpus 4): bench.py JSON lines into gpurun_out/r02_<workload>_n<N>[_<tag>].json
set -u
mkdir -p gpurun_out
run() {  # tag workload N extra...
  local tag=$1 w=$2 n=$3; shift 3
  local out=gpurun_out/r02_${w}_n${n}${tag:+_$tag}
  if [ "$n" = 1 ]; then
    timeout 900 python bench.py --workload "$w" "$@" > $out.json 2> $out.err
  else
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr=127.0.0.1 \
      --master-port=$((29500 + n)) bench.py --gpus $n --workload "$w" "$@" > $out.json 2> $out.err
  fi
  echo "$w n=$n $tag rc=$? $(python -c "import json; d=json.loads(open('$out.json').read().strip().splitlines()[-1]); print('ms', round(d['ms_per_step'],3), 'frac', round(d['step_roofline']['frac'],3), {k: round(v['avg_ms'],3) for k,v in d['kernels'].items()})" 2>/dev/null)"
}
for n in 2 4; do run "" flat7b_1bit_sync $n --steps 10 --no-cpu-baseline --no-e2e; done
run default flat7b_1bit_sync 4 --steps 10 --no-cpu-baseline
run "" flat7b_1bit 4 --steps 10 --no-cpu-baseline --no-e2e
run "" c1_1bit_1m 4 --steps 50 --no-cpu-baseline --no-e2e
for n in 2 4; do run "" tinyllama_1bit_sync $n --steps 50 --no-cpu-baseline --no-e2e; done
LIONCUB_ERRORS=deferred run deferred tinyllama_1bit_sync 4 --steps 50 --no-cpu-baseline --no-e2e
for n in 2 4; do run "" tinyllama_1bit $n --steps 50 --no-cpu-baseline --no-e2e; done
run "" gpt2s_sumsigns 4 --steps 50 --no-cpu-baseline --no-e2e
LIONCUB_ERRORS=deferred run deferred gpt2s_sumsigns 4 --steps 50 --no-cpu-baseline --no-e2e
run "" gpt2s_l1_5bit 1 --steps 50 --no-cpu-baseline --no-e2e
run "" gpt2s_l1_5bit 4 --steps 50 --no-cpu-baseline --no-e2e
run "" gpt2s_ps 4 --steps 30 --no-cpu-baseline --no-e2e
echo done
