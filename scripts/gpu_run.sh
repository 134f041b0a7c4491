mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
python -c "import torch;print(torch.cuda.get_device_name(0))" > gpurun_out/dev.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 -k "not cfg4_full" > gpurun_out/pytest1.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest1.log
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -q --timeout 850 -k "cfg4_full" > gpurun_out/pytest2.log 2>&1; echo "pytest2 rc=$?" >> gpurun_out/pytest2.log
timeout 1200 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench1.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench1.log
