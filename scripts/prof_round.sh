# Round evidence: GPU tests, full bench, launch list, ncu captures of the top kernels (one GPU)
mkdir -p gpurun_out
P=${PROF_TAG:-r01b}
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/${P}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${P}_pytest.log
timeout 900 python bench.py > gpurun_out/${P}_bench.log 2>&1; echo "rc=$?" >> gpurun_out/${P}_bench.log
timeout 300 python scripts/bench_eval.py > gpurun_out/${P}_eval.json 2> gpurun_out/${P}_eval.err
python scripts/profile_target.py lattice > gpurun_out/${P}_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lattice_measures -s 1 -c 1 -o gpurun_out/${P}_measures python scripts/profile_target.py lattice > gpurun_out/${P}_ncu_m.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lattice_table -s 32 -c 1 -o gpurun_out/${P}_table python scripts/profile_target.py lattice > gpurun_out/${P}_ncu_t.log 2>&1
python scripts/profile_target.py eval10 > gpurun_out/${P}_plain_e.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_eval -s 1 -c 1 -o gpurun_out/${P}_eval10 python scripts/profile_target.py eval10 > gpurun_out/${P}_ncu_e.log 2>&1
python scripts/profile_target.py eval16 > gpurun_out/${P}_plain_e16.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_eval -s 1 -c 1 -o gpurun_out/${P}_eval16 python scripts/profile_target.py eval16 > gpurun_out/${P}_ncu_e16.log 2>&1
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-percell > gpurun_out/${P}_plain_b.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${P}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-percell > gpurun_out/${P}_ncu_launch.log 2>&1
echo done
