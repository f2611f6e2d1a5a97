#!/bin/bash
# C5-style sweep of the ZP executor on one box (run through gpurun --gpus 4):
# schedule (ZP / DistEP), Asym-EA on/off, router skew (Zipf alpha), expert-rank capacity w.
# One JSON line per run under gpurun_out/sweep/<N>gpu_<name>.json.
set -u
mkdir -p gpurun_out/sweep
STEPS=${STEPS:-4}
run() {  # n name args...
  local n=$1 name=$2; shift 2
  local devs=$(seq -s, 0 $((n - 1)))
  CUDA_VISIBLE_DEVICES=$devs timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
    --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus $n --steps $STEPS \
    --warmup 3 ${EXTRA:-} "$@" > gpurun_out/sweep/${n}gpu_${name}.json 2> gpurun_out/sweep/${n}gpu_${name}.err
  echo "$n $name rc=$?"
}
for n in ${NS:-4 2}; do
  run $n zp_asym
  run $n zp_noasym --no-asym-ea
  run $n distep --schedule distep
  run $n zp_nccl --transport nccl
  for a in 0.5 1.0 1.5; do run $n zp_asym_skew$a --router-skew $a; done
  run $n zp_noasym_skew1.0 --no-asym-ea --router-skew 1.0
  if [ $n -ge 4 ]; then
    for w in 0.75 0.5; do run $n zp_asym_cap$w --expert-capacity $w; run $n zp_noasym_cap$w --no-asym-ea --expert-capacity $w; done
  fi
done
