# ring-depth variants with the slot-release fence (headline timing only)
mkdir -p gpurun_out
T=${TAG:-sw6}
for cfg in "HOI_RING=4" "HOI_RING=5" "HOI_RING=6" "HOI_RING=4" "HOI_RING=5"; do
  echo "== $cfg" >> gpurun_out/${T}.log
  env $cfg timeout 300 python bench.py --no-cpu-baseline --no-percell --no-cfg5 --steps 10 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); r=j['roofline']; print(round(j['ms_per_step'],3), round(r['kernel_ms'],3), round(r['table_kernel_ms'],3), 'e2e', round(j['e2e']['seconds_per_step']*1e3,2))" >> gpurun_out/${T}.log 2>&1
done
