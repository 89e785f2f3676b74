# single-GPU vote/update variants at two sizes (tests/va_microbench.py)
for n in 124439808 1100048384; do
for v in ${VARIANTS:-default i32k i512k c16 default}; do
  if [ $v = default ]; then unset LIONCUB_LIB; else export LIONCUB_LIB=$PWD/paper_2411_16462_b200/_lib/liblioncub_$v.so; fi
  echo "$v $(timeout 300 python tests/va_microbench.py --n $n --iters 50 --only ${ONLY:-vote_apply,apply_update} 2>&1 | tail -1)"
done; done
