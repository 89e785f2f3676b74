# Round measurement sweep on one 4-GPU box: bench.py JSON lines per
# workload and GPU count into gpurun_out/meas_<workload>_n<N>.json
#   gpurun --gpus 4 -- bash tests/measure_round.sh
set -u
mkdir -p gpurun_out
run() {  # workload N extra-args...
  local w=$1 n=$2; shift 2
  if [ "$n" = 1 ]; then
    timeout 900 python bench.py --workload "$w" "$@" > gpurun_out/meas_${w}_n1.json 2> gpurun_out/meas_${w}_n1.err
  else
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr=127.0.0.1 \
      --master-port=$((29500 + n)) bench.py --gpus $n --workload "$w" "$@" \
      > gpurun_out/meas_${w}_n$n.json 2> gpurun_out/meas_${w}_n$n.err
  fi
  echo "$w n=$n rc=$? $(tail -c 200 gpurun_out/meas_${w}_n$n.json | grep -o '"ms_per_step": [0-9.]*')"
}
run gpt2s_sumsigns 1
for n in 2 4; do run gpt2s_sumsigns $n --no-cpu-baseline; done
for n in 1 2 4; do run tinyllama_1bit_sync $n --no-cpu-baseline --no-e2e; done
for n in 1 2 4; do run gpt2s_l1_5bit $n --no-cpu-baseline --no-e2e; done
for n in 1 4; do run gpt2s_qinf_stoch_5bit $n --no-cpu-baseline --no-e2e; done
run c1_1bit_1m 1 --no-cpu-baseline
for n in 2 4; do run gpt2s_ps $n --no-cpu-baseline --no-e2e; done
