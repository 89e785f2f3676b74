# single-GPU vote/update kernel variants (tests/va_microbench.py)
for v in ${VARIANTS:-default m3 m4 c4m3 c4m4 c16m3 k8m3 c2m4 m3 default}; do
  if [ $v = default ]; then unset LIONCUB_LIB; else export LIONCUB_LIB=$PWD/paper_2411_16462_b200/_lib/liblioncub_$v.so; fi
  echo "$v $(timeout 300 python tests/va_microbench.py --iters 20 --only ${ONLY:-vote_apply,apply_update} 2>&1 | tail -1)"
done
