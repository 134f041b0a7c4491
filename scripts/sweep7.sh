# TopK filter variants with the slot-release fence: e2e (public API) timing
mkdir -p gpurun_out
T=${TAG:-sw7}
for cfg in "HOI_TWO_PASS_FILTER=0" "HOI_TWO_PASS_FILTER=1" "HOI_TWO_PASS_FILTER=1 HOI_PREFETCH=1" "HOI_PREFETCH=1" "HOI_TWO_PASS_FILTER=0" "HOI_TWO_PASS_FILTER=1 HOI_PREFETCH=1"; do
  echo "== $cfg" >> gpurun_out/${T}.log
  env $cfg timeout 300 python bench.py --no-cpu-baseline --no-percell --no-cfg5 --steps 5 --e2e-steps 5 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); r=j['roofline']; print(round(j['ms_per_step'],3), round(r['kernel_ms'],3), 'e2e', round(j['e2e']['seconds_per_step']*1e3,2))" >> gpurun_out/${T}.log 2>&1
done
