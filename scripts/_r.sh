mkdir -p gpurun_out
T=${TAG:-r}
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -k "${KSEL:-lattice or cfg4 or cfg3 or topk or cfg1 or cfg2 or sampled or shard or identity or fullrow}" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
for i in 1 2; do timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-percell --no-cfg5 --steps 10 > gpurun_out/${T}_bench$i.log 2>&1; done
if [ -n "$NCU" ]; then python scripts/profile_target.py lattice > gpurun_out/${T}_plainl.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lattice -s 3 -c 3 -o gpurun_out/${T}_lattice python scripts/profile_target.py lattice > gpurun_out/${T}_ncul.log 2>&1; fi
