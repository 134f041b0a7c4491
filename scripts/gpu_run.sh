mkdir -p gpurun_out
python scripts/profile_target.py fused > gpurun_out/plain_fused.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lattice_fused -s 1 -c 1 -o gpurun_out/prof_fused python scripts/profile_target.py fused > gpurun_out/ncu_fused.log 2>&1
echo done
