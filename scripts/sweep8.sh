# filtered stencil: 6-slot ring without neighbour-sum buffers vs the 4-slot ring (e2e TopK)
mkdir -p gpurun_out
T=${TAG:-sw10}
for cfg in "HOI_FILTER_RING6=1" "HOI_FILTER_RING6=0" "HOI_FILTER_RING6=1 HOI_TWO_PASS_FILTER=1" "HOI_FILTER_RING6=0 HOI_TWO_PASS_FILTER=1" "HOI_FILTER_RING6=1" "HOI_FILTER_RING6=0"; do
  echo "== $cfg" >> gpurun_out/${T}.log
  env $cfg timeout 300 python bench.py --no-cpu-baseline --no-percell --no-cfg5 --steps 3 --e2e-steps 5 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('e2e', round(j['e2e']['seconds_per_step']*1e3,2))" >> gpurun_out/${T}.log 2>&1
done
