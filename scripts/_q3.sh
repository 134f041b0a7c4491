mkdir -p gpurun_out
T=${TAG:-q3}
python scripts/bw_probe.py > gpurun_out/${T}_bw.json 2>&1
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -k "objective or optim or greedy or anneal or copula or cov" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
python scripts/profile_target.py copula5 > gpurun_out/${T}_plainc.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -s 5 -c 5 -o gpurun_out/${T}_copula5 python scripts/profile_target.py copula5 > gpurun_out/${T}_ncuc.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-percell --steps 5 > gpurun_out/${T}_bench.log 2>&1
