mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest.log
timeout 1200 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/plain_launch.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
python scripts/profile_target.py lattice > gpurun_out/plain_lattice.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lattice -s 2 -c 2 -o gpurun_out/prof_lattice python scripts/profile_target.py lattice > gpurun_out/ncu_lattice.log 2>&1
python scripts/profile_target.py eval10 > gpurun_out/plain_eval10.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_eval -s 1 -c 1 -o gpurun_out/prof_eval10 python scripts/profile_target.py eval10 > gpurun_out/ncu_eval10.log 2>&1
echo done
