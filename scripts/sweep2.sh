mkdir -p gpurun_out
T=${TAG:-sw}
timeout 600 env HOI_PIPE=1 python -m pytest tests -m gpu -q -x --timeout 500 -k "lattice or cfg4 or cfg3 or topk or cfg1 or cfg2 or sampled" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
for cfg in "HOI_PIPE=0" "HOI_PIPE=1" "HOI_PIPE=1 HOI_PIPE_WB=17" "HOI_PIPE=1 HOI_PIPE_WB=15" "HOI_PIPE=1 HOI_STENCIL_PER_SM=2" "HOI_PIPE=1 HOI_TABLE_NW=8 HOI_STENCIL_PER_SM=2" "HOI_PIPE=1 HOI_STENCIL_PER_SM=4"; do
  echo "== $cfg" >> gpurun_out/${T}.log
  env $cfg timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-percell --steps 10 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); r=j['roofline']; print(round(j['ms_per_step'],3), round(r['kernel_ms'],3), round(r['table_kernel_ms'],3))" >> gpurun_out/${T}.log 2>&1
done
