mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -x -k "lattice or cfg4 or cfg3 or topk" > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest.log
timeout 300 python scripts/e2e_profile.py > gpurun_out/e2e_profile.log 2>&1
python scripts/profile_target.py lattice > gpurun_out/plain_lattice.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lattice_measures -s 1 -c 1 -o gpurun_out/prof_lattice3 python scripts/profile_target.py lattice > gpurun_out/ncu_lattice.log 2>&1
echo done
