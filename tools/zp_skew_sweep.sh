set -u
mkdir -p gpurun_out/sweep2
run() { local n=$1 name=$2; shift 2; local devs=$(seq -s, 0 $((n - 1)))
  CUDA_VISIBLE_DEVICES=$devs timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus $n --steps 4 --warmup 3 "$@" > gpurun_out/sweep2/${n}gpu_${name}.json 2> gpurun_out/sweep2/${n}gpu_${name}.err; echo "$n $name rc=$?"; }
for n in 4 2; do
  for a in 0.5 1.0 1.5; do run $n zp_asym_skew$a --router-skew $a; done
  run $n zp_noasym_skew1.0 --no-asym-ea --router-skew 1.0
done
