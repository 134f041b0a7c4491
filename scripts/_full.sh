mkdir -p gpurun_out
T=${TAG:-f}
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
timeout 300 python __graft_entry__.py > gpurun_out/${T}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_smoke.log
timeout 900 python bench.py > gpurun_out/${T}_bench.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_bench.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${T}_ref.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_ref.log
HOI_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 1 --no-cfg5 > gpurun_out/${T}_dist.log 2> gpurun_out/${T}_dist.err; echo "rc=$?" >> gpurun_out/${T}_dist.log
