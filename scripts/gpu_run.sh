mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -x -k "lattice or fused or cfg4 or cfg3 or topk" > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest.log
timeout 600 python bench.py --engine 2 --no-cpu-baseline --no-e2e --steps 10 > gpurun_out/bench_e2.log 2>&1; echo "rc=$?" >> gpurun_out/bench_e2.log
python scripts/profile_target.py lattice > gpurun_out/plain_lattice.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lattice_measures -s 8 -c 1 -o gpurun_out/prof_lattice5 python scripts/profile_target.py lattice > gpurun_out/ncu_lattice.log 2>&1
echo done
