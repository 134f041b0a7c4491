mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -x -k "lattice or fused or cfg4 or cfg3 or topk" > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest.log
timeout 600 python bench.py --engine 2 --no-cpu-baseline --steps 10 > gpurun_out/bench_e2.log 2>&1; echo "rc=$?" >> gpurun_out/bench_e2.log
echo done
