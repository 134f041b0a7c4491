# ncu captures of the current kernels (one GPU); run under gpurun
mkdir -p gpurun_out
P=${PROF_TAG:-base}
python scripts/profile_target.py lattice > gpurun_out/plain_${P}.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lattice_measures -s 1 -c 1 -o gpurun_out/${P}_measures python scripts/profile_target.py lattice > gpurun_out/ncu_${P}_m.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lattice_table -s 1 -c 1 -o gpurun_out/${P}_table python scripts/profile_target.py lattice > gpurun_out/ncu_${P}_t.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_eval -s 1 -c 1 -o gpurun_out/${P}_eval10 python scripts/profile_target.py eval10 > gpurun_out/ncu_${P}_e.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${P}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_${P}_launch.log 2>&1
echo done
