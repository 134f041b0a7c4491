mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -x > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest.log
timeout 300 python scripts/e2e_profile.py > gpurun_out/e2e_profile.log 2>&1
timeout 1200 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
python scripts/profile_target.py lattice > gpurun_out/plain_lattice.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lattice -s 2 -c 2 -o gpurun_out/prof_lattice2 python scripts/profile_target.py lattice > gpurun_out/ncu_lattice.log 2>&1
echo done
