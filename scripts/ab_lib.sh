# A/B timing of two builds of libhoib200.so on one box: $1 = alternate .so;
# runs the lattice-only bench line alternately (new, old, new, old).
L=paper_2501_03381_b200/_lib/libhoib200.so
cp $L /tmp/lib_new.so
for r in ${ROUNDS:-1 2}; do
  for v in new old; do
    if [ $v = new ]; then cp /tmp/lib_new.so $L; else cp $1 $L; fi
    touch $L
    timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-percell --no-cfg5 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readline()); r=d['roofline']; print('$v', 'step', round(d['ms_per_step'],3), 'table', round(r['table_kernel_ms'],3), 'passes', round(r['kernel_ms'],3), 'clk', d['clocks']['sm_mhz'])"
  done
done
cp /tmp/lib_new.so $L
