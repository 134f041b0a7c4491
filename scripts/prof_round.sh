# Round evidence: GPU tests, smoke, full bench, reference arm, launch list,
# ncu captures of the top kernels (one GPU, one process at a time)
mkdir -p gpurun_out
P=${PROF_TAG:-r02}
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/${P}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${P}_pytest.log
timeout 300 python __graft_entry__.py > gpurun_out/${P}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${P}_smoke.log
timeout 900 python bench.py > gpurun_out/${P}_bench.log 2>&1; echo "rc=$?" >> gpurun_out/${P}_bench.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${P}_ref.log 2>&1; echo "rc=$?" >> gpurun_out/${P}_ref.log
python scripts/bw_probe.py > gpurun_out/${P}_bw.json 2>&1
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-percell --no-cfg5 > gpurun_out/${P}_plain_b.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/${P}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-percell --no-cfg5 > gpurun_out/${P}_ncu_launch.log 2>&1
python scripts/profile_target.py lattice > gpurun_out/${P}_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lattice -s 3 -c 3 -o gpurun_out/${P}_lattice python scripts/profile_target.py lattice > gpurun_out/${P}_ncu_l.log 2>&1
python scripts/profile_target.py eval10 > gpurun_out/${P}_plain_e.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_eval -s 1 -c 1 -o gpurun_out/${P}_eval10 python scripts/profile_target.py eval10 > gpurun_out/${P}_ncu_e.log 2>&1
python scripts/profile_target.py copula5 > gpurun_out/${P}_plain_c.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -s 6 -c 6 -o gpurun_out/${P}_copula5 python scripts/profile_target.py copula5 > gpurun_out/${P}_ncu_c.log 2>&1
echo done
