# GPU test run: $1 = pytest selection (default: all gpu tests), logs to gpurun_out/
mkdir -p gpurun_out
T=${TAG:-t}
timeout ${TMO:-1500} python -m pytest ${SEL:-tests} -m gpu -q --timeout 900 -x ${PYARGS} > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
