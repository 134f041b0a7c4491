# A/B of scripts/shard_times.py (per-rank shard bounds) for two builds: $1 = alternate .so
L=paper_2501_03381_b200/_lib/libhoib200.so
cp $L /tmp/lib_new.so
for v in new old; do
  if [ $v = new ]; then cp /tmp/lib_new.so $L; else cp $1 $L; fi
  touch $L
  echo "$v: $(timeout 600 python scripts/shard_times.py 2>/dev/null | tail -1)"
done
cp /tmp/lib_new.so $L
