# The driver's scaling sequence on one 4-GPU box: both arms at N = 1, 2, 4, launched as the driver
# launches them (torchrun for N > 1), one JSON line each into gpurun_out/scale/.
set -u
mkdir -p gpurun_out/scale
for n in 1 2 4; do
  for impl in reference ours; do
    if [ "$n" = 1 ]; then
      timeout 900 python bench.py --impl $impl --gpus 1 --steps 10 --warmup 3 > gpurun_out/scale/${impl}_$n.json 2> gpurun_out/scale/${impl}_$n.err
    else
      timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
        --master-port $((29700 + n)) bench.py --impl $impl --gpus $n --steps 10 --warmup 3 \
        > gpurun_out/scale/${impl}_$n.json 2> gpurun_out/scale/${impl}_$n.err
    fi
    echo "$impl $n rc=$?"
  done
done
