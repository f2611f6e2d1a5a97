# BASELINE C5 sweep on one 4-GPU box (final tree): router skew (Zipf alpha) and per-rank expert
# capacity weights at 2 + 2 and 1 + 1, plus the 3 + 1 split. One JSON line per run in
# gpurun_out/c5/; tools/sweep_table.py gpurun_out/c5 renders the table.
set -u
mkdir -p gpurun_out/c5
run() { local n=$1 name=$2; shift 2; local devs=$(seq -s, 0 $((n - 1)))
  CUDA_VISIBLE_DEVICES=$devs timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
    --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus $n --steps 4 --warmup 3 \
    --no-stack-reference "$@" > gpurun_out/c5/${n}gpu_${name}.json 2> gpurun_out/c5/${n}gpu_${name}.err
  echo "$n $name rc=$?"; }
run 4 base
for a in 0.5 1.0 1.5; do run 4 skew$a --router-skew $a; done
run 4 skew1.0_contiguous --router-skew 1.0 --no-balanced-placement
run 4 cap_1_0.75 --expert-capacity 1,0.75
run 4 cap_1_0.5 --expert-capacity 1,0.5
run 4 split3+1 --attention-ranks 3
run 2 base
run 2 skew1.0 --router-skew 1.0
run 2 cap_0.5 --expert-capacity 0.5
