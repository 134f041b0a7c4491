mkdir -p gpurun_out
T=${TAG:-q2}
python scripts/ab_full.py > gpurun_out/${T}_ab.json 2> gpurun_out/${T}_ab.err
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -k "copula or cov or rank or cfg1 or cfg4_full or helpers or ref_copula or acceptance" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
python scripts/cfg5_topk.py > gpurun_out/${T}_topk.json 2>&1
