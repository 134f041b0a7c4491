mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -k "copula or rank or cov or cfg or ref_copula or helpers or acceptance" > gpurun_out/c1_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/c1_pytest.log
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-percell --no-cfg5 > /dev/null 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/c1_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-percell --no-cfg5 > gpurun_out/c1_ncu.log 2>&1
