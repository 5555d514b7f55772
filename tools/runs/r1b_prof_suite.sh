tr() { python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 "${@:3}"; }
for n in 2 4; do
  for wl in lm1b_sparse lm1b; do
    echo "== n=$n $wl"
    timeout 200 bash -c "$(declare -f tr); tr $n $((29600+n)) tools/prof_multi.py $wl" 2>&1 | grep '^{'
  done
  echo "== n=$n spans lm1b_sparse"
  timeout 200 bash -c "$(declare -f tr); tr $n $((29610+n)) tools/span_multi.py lm1b_sparse" 2>&1 | grep '^{'
  echo "== n=$n spans table"
  timeout 200 bash -c "$(declare -f tr); tr $n $((29620+n)) tools/span_multi.py table" 2>&1 | grep '^{'
done
