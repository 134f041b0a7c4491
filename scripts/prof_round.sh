# Round evidence: GPU tests, full bench, launch list, ncu captures of the top kernels (one GPU)
mkdir -p gpurun_out
P=${PROF_TAG:-r01l}
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/${P}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${P}_pytest.log
timeout 300 python __graft_entry__.py > gpurun_out/${P}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${P}_smoke.log
timeout 900 python bench.py > gpurun_out/${P}_bench.log 2>&1; echo "rc=$?" >> gpurun_out/${P}_bench.log
timeout 300 python scripts/bench_eval.py > gpurun_out/${P}_eval.json 2> gpurun_out/${P}_eval.err
python scripts/profile_target.py lattice > gpurun_out/${P}_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lattice -s 3 -c 3 -o gpurun_out/${P}_lattice python scripts/profile_target.py lattice > gpurun_out/${P}_ncu_l.log 2>&1
python scripts/profile_target.py eval10 > gpurun_out/${P}_plain_e.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_eval -s 1 -c 1 -o gpurun_out/${P}_eval10 python scripts/profile_target.py eval10 > gpurun_out/${P}_ncu_e.log 2>&1
python scripts/profile_target.py eval20 > gpurun_out/${P}_plain_e20.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_eval -s 1 -c 1 -o gpurun_out/${P}_eval20 python scripts/profile_target.py eval20 > gpurun_out/${P}_ncu_e20.log 2>&1
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-percell --no-cfg5 > gpurun_out/${P}_plain_b.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/${P}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-percell --no-cfg5 > gpurun_out/${P}_ncu_launch.log 2>&1
echo done
