# env-knob sweep of the stencil kernel (headline timing only)
mkdir -p gpurun_out
T=${TAG:-sw}
timeout 600 python -m pytest tests -m gpu -q -x --timeout 500 -k "lattice or cfg4 or cfg3 or topk or fused or cfg1 or cfg2 or sampled" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
for cfg in ${CFGS:-"HOI_RING=6" "HOI_RING=4" "HOI_RING=6 HOI_NEAR_BITS=20" "HOI_RING=4 HOI_NEAR_BITS=20" "HOI_RING=4 HOI_NEAR_BITS=20 HOI_OWN_LAST=1"}; do
  echo "== $cfg" >> gpurun_out/${T}.log
  env $cfg timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-percell --steps 10 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); r=j['roofline']; print(round(j['ms_per_step'],3), round(r['kernel_ms'],3), round(r['table_kernel_ms'],3))" >> gpurun_out/${T}.log 2>&1
done
