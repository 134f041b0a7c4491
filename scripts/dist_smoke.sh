# Smoke test of bench.py's multi-rank path on a ONE-GPU box: two ranks
# share cuda:0 over gloo (correctness of the N > 1 code path only; the
# numbers it prints are not a measurement).
mkdir -p gpurun_out
HOI_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 1 \
  > gpurun_out/dist_smoke.log 2> gpurun_out/dist_smoke.err
echo "rc=$?" >> gpurun_out/dist_smoke.log
