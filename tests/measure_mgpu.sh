# Multi-GPU measurement pass on one box (gpurun --gpus N): bench.py JSON lines
# into gpurun_out/mg_<workload>_n<N>.json, then the multi-GPU parity tests.
#   gpurun --gpus 4 -- bash tests/measure_mgpu.sh "flat7b_1bit_sync tinyllama_1bit_sync" "2 4" [pytest]
set -u
mkdir -p gpurun_out
WL=${1:-"flat7b_1bit_sync tinyllama_1bit_sync gpt2s_sumsigns"}
NS=${2:-"2 4"}
for w in $WL; do
  for n in $NS; do
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr=127.0.0.1 \
      --master-port=$((29500 + n)) bench.py --gpus $n --workload "$w" --steps ${STEPS:-20} --warmup 5 \
      --no-cpu-baseline ${EXTRA:-} > gpurun_out/mg_${w}_n$n.json 2> gpurun_out/mg_${w}_n$n.err
    echo "$w n=$n rc=$? $(python -c "import json,sys; d=json.loads(open('gpurun_out/mg_${w}_n$n.json').read().strip().splitlines()[-1]); print('ms', round(d['ms_per_step'],3), 'step_frac', round(d['step_roofline']['frac'],3), 'dom', d['roofline']['kernel'], round(d['roofline']['frac'],3))" 2>/dev/null)"
  done
done
if [ "${3:-}" = "pytest" ]; then
  timeout 1500 python -m pytest tests/test_multigpu.py -q --timeout 600 > gpurun_out/mg_pytest.log 2>&1
  echo "pytest rc=$?"; tail -3 gpurun_out/mg_pytest.log
fi
