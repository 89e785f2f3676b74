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
  echo "$w n=$n rc=$?"
}
run gpt2s_sumsigns 1
for n in 2 4; do run gpt2s_sumsigns $n --no-cpu-baseline; done
for n in 1 2 4; do run tinyllama_1bit_sync $n --no-cpu-baseline --no-e2e; done
for n in 1 2 4; do run gpt2s_l1_5bit $n --no-cpu-baseline --no-e2e; done
for n in 1 4; do run gpt2s_qinf_stoch_5bit $n --no-cpu-baseline --no-e2e; done
run c1_1bit_1m 1 --no-cpu-baseline
run gpt2s_1bit_syncall 4 --no-cpu-baseline --no-e2e
for n in 2 4; do run gpt2s_ps $n --no-cpu-baseline --no-e2e; done
# reference arm (CPU port) on the default workload
timeout 600 python bench.py --impl reference > gpurun_out/meas_reference_n1.json 2> gpurun_out/meas_reference_n1.err
# kernel launch list of the default bench and ncu of the norm pass
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/launches_default.csv 2>/dev/null
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none -k regex:k_l1 --csv python tests/profile_kernels.py --n 1048576 --reps 1 > gpurun_out/ncu_l1_final.csv 2>/dev/null
echo done
