#!/bin/bash
# Builder-side multi-GPU bench sweep (gpurun --gpus N): one JSON line per
# (nproc, P x D, dispatch) into gpurun_out/$TAG_bench_*.txt.
# usage: tools/multi_bench.sh TAG "nproc:PxD:dispatch[:extra]" ...
TAG=$1; shift
mkdir -p gpurun_out
for spec in "$@"; do
  IFS=: read -r n pd disp extra <<< "$spec"
  out=gpurun_out/${TAG}_bench_${n}g_${pd}_${disp}.txt
  if [ "$n" = "1" ]; then
    timeout 900 python bench.py --gpus 1 --pd "$pd" --dispatch "$disp" --steps 8 --warmup 3 $extra > "$out" 2>&1
  else
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node="$n" --master-addr=127.0.0.1 \
      --master-port=$((29600 + RANDOM % 1000)) bench.py --gpus "$n" --pd "$pd" --dispatch "$disp" \
      --steps 8 --warmup 3 $extra > "$out" 2>&1
  fi
  echo "== $spec rc=$?"; grep -o '"value": [0-9.]*\|"bubble": {[^}]*}' "$out" | head -3
done
