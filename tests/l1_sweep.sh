# L1 norm pass variants on the GPT-2 layout at P=1 (bench.py kernel timers)
for v in ${VARIANTS:-default lm5 lm6 lm3 default}; do
  if [ $v = default ]; then unset LIONCUB_LIB; else export LIONCUB_LIB=$PWD/paper_2411_16462_b200/_lib/liblioncub_$v.so; fi
  timeout 300 python bench.py --workload gpt2s_l1_5bit --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/l1.json 2> gpurun_out/l1.err
  python -c "import json; d=json.loads(open('gpurun_out/l1.json').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],3), {k: round(v['avg_ms'],3) for k,v in d['kernels'].items()})"
done
