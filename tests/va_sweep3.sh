# single-GPU vote/update variants at 1.1B and 124M, P=4 and P=2 (tests/va_microbench.py)
for v in ${VARIANTS:-default inl m3 inlm3 default}; do
  if [ $v = default ]; then unset LIONCUB_LIB; else export LIONCUB_LIB=$PWD/paper_2411_16462_b200/_lib/liblioncub_$v.so; fi
  a=$(timeout 300 python tests/va_microbench.py --only vote_apply 2>&1 | tail -1 | python -c "import json,sys; print(json.loads(sys.stdin.read())['vote_apply']['ms'])")
  b=$(timeout 300 python tests/va_microbench.py --P 2 --only vote_apply 2>&1 | tail -1 | python -c "import json,sys; print(json.loads(sys.stdin.read())['vote_apply']['ms'])")
  c=$(timeout 300 python tests/va_microbench.py --n 124439808 --iters 50 --only vote_apply 2>&1 | tail -1 | python -c "import json,sys; print(json.loads(sys.stdin.read())['vote_apply']['ms'])")
  echo "$v 1.1B/P4 $a 1.1B/P2 $b 124M/P4 $c"
done
