# quick GPU iteration: lattice parity tests + headline timing (no CPU leg, no e2e)
mkdir -p gpurun_out
T=${TAG:-q}
timeout 600 python -m pytest tests -m gpu -q -x --timeout 500 -k "${KSEL:-lattice or cfg4 or cfg3 or topk or fused or cfg1 or cfg2 or sampled}" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 10 > gpurun_out/${T}_bench.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_bench.log
