# pass 2: partial-sum job first vs after the neighbours (headline step)
mkdir -p gpurun_out
T=${TAG:-sw16}
for cfg in "HOI_EXTRA_FIRST=1" "HOI_EXTRA_FIRST=0" "HOI_EXTRA_FIRST=1" "HOI_EXTRA_FIRST=0"; do
  echo "== $cfg" >> gpurun_out/${T}.log
  env $cfg timeout 300 python bench.py --no-cpu-baseline --no-percell --no-cfg5 --no-e2e --steps 10 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); r=j['roofline']; print(round(j['ms_per_step'],3), round(r['kernel_ms'],3), round(r['table_kernel_ms'],3))" >> gpurun_out/${T}.log 2>&1
done
